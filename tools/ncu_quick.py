"""Quick look at an ncu report: duration, pipe utilisation, stall reasons, top
SASS opcodes by stall samples (measurement tooling)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "smsp__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__registers_per_thread"]
for k in want:
    if k in h:
        print(k, v[h.index(k)])
stalls = [(k, v[i]) for i, k in enumerate(h) if k.startswith("smsp__average_warp_latency_issue_stalled_") or
          k.startswith("smsp__pcsamp_warps_issue_stalled_")]
st = []
for k, x in stalls:
    try:
        st.append((float(x), k))
    except ValueError:
        pass
for x, k in sorted(st, reverse=True)[:12]:
    print(f"  {k} {x}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(src)))
hh = r[1]
ix, sc, ss = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
agg = {}
for row in r[2:]:
    if len(row) <= ix:
        continue
    parts = row[sc].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    op = op.split(".")[0]
    try:
        agg.setdefault(op, [0, 0])
        agg[op][0] += float(row[ix] or 0)
        agg[op][1] += float(row[ss] or 0)
    except ValueError:
        pass
tot = sum(a[1] for a in agg.values()) or 1
print("opcode  executed  stall-samples%")
for op, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"  {op:8s} {n:12.0f} {100*s/tot:6.1f}")
