"""GPU roofline model (include/lbg.h lbg_characterize / place / classify and the
machine-profile text format) against the reference's own roofline.cpp
(compiled from its sources in oracle/_ref), and the measured B200 profile."""
import json
import os

import numpy as np
import pytest

# B200 ladder as measured (profiles/r01_fp64_peaks.json, MEASURED_PEAKS.json):
# SMEM 36.9 TB/s, L2 15.4 TB/s, HBM 6.47 TB/s, PCIe ~55 GB/s
B200 = ("b200", 37040.0, [36895.5, 15363.8, 6465.2, 55.0], [233472, 132120576, 191514411008])
CPU = ("i9-13980HX", 128.0, [250.0, 150.0, 100.0, 80.0], [48 * 1024, 2 * 1024 * 1024, 36 * 1024 * 1024])


@pytest.mark.parametrize("prof", [B200, CPU])
@pytest.mark.parametrize("d", [1, 2, 3, 5, 9, 16, 27, 40, 81])
def test_characterize_place_classify_match_reference(lbg, reference, prof, d):
    m = lbg.machine_profile(*prof)
    k = lbg.place(lbg.characterize(d), m)
    c = lbg.classify(k, m)
    want = reference.roofline(d, prof[1], prof[2], prof[3])
    assert (k.flops, k.bytes, k.placement) == (want["flops"], want["bytes"], want["placement"])
    assert k.ai == want["ai"] and c["attainable_gflops"] == want["attainable_gflops"]
    assert (c["bound"] == "compute_bound") == (want["bound"] == 1)


def test_profile_text_round_trips_through_the_reference(lbg, reference):
    m = lbg.machine_profile(*B200)
    text = lbg.write_machine_profile(m)
    assert text == reference.write_profile(*B200)
    back = reference.read_profile(text, "b200")  # the reference's parser loads a B200 profile
    assert back["capacity_bytes"] == B200[3]
    ours = lbg.read_machine_profile(text, "b200")
    assert list(ours.capacity_bytes) == B200[3] and ours.name == b"b200"
    assert np.allclose(list(ours.bandwidth_gbs), back["bandwidth_gbs"], rtol=0, atol=0)


@pytest.mark.parametrize("text,exc", [
    ("peak_gflops = 1\n", RuntimeError),                                  # missing keys
    ("peak_gflops 1\n", RuntimeError),                                    # no '='
    ("peak_gflops = x\n", RuntimeError),                                  # bad number
    ("peak_gflops = 1\npeak_gflops = 2\n", RuntimeError),                 # duplicate
    ("peak_gflops=1\nbw_l1=4\nbw_l2=3\nbw_l3=2\nbw_dram=1\ncap_l1=1\ncap_l2=2\ncap_l3=3\nfoo=1\n", RuntimeError),
    ("peak_gflops=1\nbw_l1=4\nbw_l2=3\nbw_l3=2\nbw_dram=1\ncap_l1=1\ncap_l2=2\ncap_l3=2.5\n", RuntimeError),
    ("peak_gflops=1\nbw_l1=1\nbw_l2=3\nbw_l3=2\nbw_dram=1\ncap_l1=1\ncap_l2=2\ncap_l3=3\n", ValueError),
    ("peak_gflops=1\nbw_l1=4\nbw_l2=3\nbw_l3=2\nbw_dram=1\ncap_l1=3\ncap_l2=2\ncap_l3=3\n", ValueError),
])
def test_profile_errors_like_reference(lbg, reference, text, exc):
    with pytest.raises(exc):
        lbg.read_machine_profile(text)
    with pytest.raises(exc):
        reference.read_profile(text)


def test_classify_requires_placement(lbg):
    with pytest.raises(ValueError):
        lbg.classify(lbg.characterize(3), lbg.machine_profile(*B200))
    with pytest.raises(ValueError):
        lbg.characterize(0)


@pytest.mark.gpu
def test_measured_b200_profile(lbg, reference):
    m = lbg.measure_machine_profile()
    d = m.as_dict()
    bw = d["bandwidth_gbs"]
    assert bw[0] > bw[1] > bw[2] > bw[3] > 0  # the ladder is strictly ordered (validate_profile)
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else {}
    if "hbm_gbs" in peaks:
        assert abs(bw[2] / peaks["hbm_gbs"] - 1) < 0.25
    assert 25000 < d["peak_gflops"] < 45000
    text = lbg.write_machine_profile(m)
    reference.read_profile(text, "b200")  # loadable by the reference's tool
    for dim, level in ((3, 0), (9, 0), (27, 1)):
        assert lbg.place(lbg.characterize(dim), m).placement == level
