"""Summarise an LBG_TILED_TRACE dump of the tiled stepping kernel (measurement
only): per step, the spread of CTA start times, each CTA's consumer time (start
-> its last consumer warp done) and the barrier wait (last warp done -> next
step start)."""
import sys
import numpy as np

raw = open(sys.argv[1], "rb").read()
grid, slots, steps = np.frombuffer(raw[:12], np.int32)
t = np.frombuffer(raw[12:], np.uint64).reshape(64, grid, slots)[:steps].astype(np.float64)
t -= t[0, :, 0].min()
start = t[:, :, 0]
done = t[:, :, 1:slots - 1].max(axis=2)
prod = t[:, :, slots - 1]
s = slice(2, steps - 1)
step_len = np.diff(start.min(axis=1))[s.start:s.stop - 1]
comp = (done - start)[s]
wait = (start[1:] - done[:-1])[s.start:s.stop - 1]
print(f"grid {grid}, steps traced {steps}")
print(f"step period (us): mean {step_len.mean()/1e3:.2f}  min {step_len.min()/1e3:.2f}  max {step_len.max()/1e3:.2f}")
print(f"start skew across CTAs (us): mean {(start.max(1)-start.min(1))[s].mean()/1e3:.2f}")
print(f"consumer time per CTA (us): mean {comp.mean()/1e3:.2f}  max-over-CTAs mean {comp.max(1).mean()/1e3:.2f}  "
      f"min-over-CTAs mean {comp.min(1).mean()/1e3:.2f}")
print(f"barrier wait (us): mean {wait.mean()/1e3:.2f}  for the last CTA {(start[1:].min(1)-done[:-1].max(1))[s.start:s.stop-1].mean()/1e3:.2f}")
print(f"producer done - start (us): mean {(prod-start)[s].mean()/1e3:.2f}")
last = comp.argmax(axis=1)
print("slowest CTAs per step:", last[:12])
