"""Text formats (host only): the 17-digit matrix interchange format and model
files, checked against the reference's own lb::write_matrix / lb::read_model
(compiled from /root/reference by oracle/Makefile)."""
import ctypes as C

import numpy as np
import pytest

AD_MODEL = """# two-level amplitude damping written for this test
dim = 2

hamiltonian =
complex-matrix 2 2
0 0
0 0
0 0
1 0

collapse =
complex-matrix 2 2
0 0
0.5 0
0 0
0 0
"""


def ref_read_model(reference, text):
    L = reference.lib
    L.ref_read_model.argtypes = [C.c_char_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t]
    d, k = C.c_size_t(), C.c_size_t()
    reference._rc(L.ref_read_model(text.encode(), C.byref(d), C.byref(k), None, None, 0), "read_model")
    h = np.zeros((d.value, d.value), np.complex128)
    ops = np.zeros((max(k.value, 1), d.value, d.value), np.complex128)
    dp = C.POINTER(C.c_double)
    reference._rc(L.ref_read_model(text.encode(), C.byref(d), C.byref(k), h.ctypes.data_as(dp),
                                   ops.ctypes.data_as(dp), k.value), "read_model")
    return h, ops[: k.value]


def test_matrix_round_trip_is_bit_exact(lbg, reference):
    rng = np.random.default_rng(4)
    a = rng.standard_normal((5, 3)) * 10.0 ** rng.integers(-300, 300, (5, 3)) + 1j * rng.standard_normal((5, 3))
    text = lbg.write_matrix(a)
    assert np.array_equal(lbg.read_matrix(text), a)
    L = reference.lib
    L.ref_write_matrix.argtypes = [C.POINTER(C.c_double), C.c_size_t, C.c_size_t, C.c_char_p, C.c_size_t,
                                   C.POINTER(C.c_size_t)]
    n = C.c_size_t()
    a = np.ascontiguousarray(a)
    buf = C.create_string_buffer(len(text) + 16)
    reference._rc(L.ref_write_matrix(a.ctypes.data_as(C.POINTER(C.c_double)), 5, 3, buf, len(buf), C.byref(n)),
                  "write_matrix")
    assert buf.value.decode() == text  # identical bytes to the reference writer


def test_read_model_matches_reference(lbg, reference):
    for text in (AD_MODEL, "preset = transmon\n", "preset = transmon\nt1 = 5e4\ntphi = inf\n",
                 "# comment\npreset = transmon\nanharmonicity = -1.88\ndrive_amp = 0.12\n"):
        h, ops = lbg.read_model(text)
        hr, opsr = ref_read_model(reference, text)
        assert np.array_equal(h, hr)
        assert np.array_equal(ops, opsr)


@pytest.mark.parametrize("text,exc", [
    ("dim = 2\n", RuntimeError),                       # missing hamiltonian
    ("preset = qutrit\n", RuntimeError),               # unknown preset
    ("dim = 2\nfoo = 1\n", RuntimeError),              # unknown key
    ("dim = x\n", RuntimeError),                       # bad number
    ("preset = transmon\ndim = 3\n", RuntimeError),    # preset excludes dim
    ("dim = 2\nhamiltonian =\ncomplex-matrix 2 2\n0 0\n1 0\n0 0\n0 0\n", ValueError),  # not Hermitian
])
def test_read_model_errors(lbg, text, exc):
    with pytest.raises(exc):
        lbg.read_model(text)


def test_model_file_runs_through_the_pipeline_shapes(lbg):
    h, ops = lbg.read_model(AD_MODEL)
    assert h.shape == (2, 2) and ops.shape == (1, 2, 2)
    assert ops[0, 0, 1] == 0.5
