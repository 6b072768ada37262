"""Dev tool: timeline of the fused fp16 kernel (TCBF_TRACE) on the radio shape -> per-tile MMA /
epilogue intervals and per-unit conversion waits, summarised over CTAs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_03269_b200 as tcbf
import synth
M, N, K, B = 1024, 1024, 256, 256
plan = tcbf.Plan(M, N, K, B, "f16")
wp = plan.pack(tcbf.WEIGHTS, synth.generate_device("phase", 1, 0, B, M, K))
x = synth.generate_device("adc", 1, 1, B, K, N)
out = plan.alloc_output()
for _ in range(3):
    plan.beamform_raw(wp, x, out=out)
torch.cuda.synchronize()
path = "/tmp/fused_trace.bin"
os.environ["TCBF_TRACE"] = path
plan.beamform_raw(wp, x, out=out)
torch.cuda.synchronize()
del os.environ["TCBF_TRACE"]
t = np.fromfile(path, dtype=np.uint64).reshape(-1, 1024).astype(np.int64)
t0 = t[t > 0].min()
nc = t.shape[0]
tiles = t[:, :512].reshape(nc, 128, 4)
units = t[:, 512:].reshape(nc, 128, 4)
ok = (tiles > 0).all(-1)
tt = np.where(tiles > 0, tiles - t0, 0) / 1e3  # us
end = tt[..., 3][ok].max()
print(f"kernel span {end:.1f} us, tiles per CTA {ok.sum(1).mean():.1f}")
mma = (tt[..., 1] - tt[..., 0])[ok]
epi = (tt[..., 3] - tt[..., 2])[ok]
gap = (tt[..., 2] - tt[..., 1])[ok]
print(f"per tile: MMA issue span {np.median(mma):.2f} us (mean {mma.mean():.2f}), epilogue {np.median(epi):.2f} us "
      f"(mean {epi.mean():.2f}), tfull->epi {np.median(gap):.2f}")
# MMA start-to-start interval
st = tt[..., 0]
d = np.diff(st, axis=1)[ok[:, 1:] & ok[:, :-1]]
print(f"MMA tile start interval: median {np.median(d):.2f} us mean {d.mean():.2f}")
es = tt[..., 2]
d = np.diff(es, axis=1)[ok[:, 1:] & ok[:, :-1]]
print(f"epilogue tile start interval: median {np.median(d):.2f} us mean {d.mean():.2f}")
uk = (units > 0).all(-1)
ut = np.where(units > 0, units - t0, 0) / 1e3
w = (ut[..., 1] - ut[..., 0])[uk]
print(f"per unit: MMA wait for B block 0: median {np.median(w):.2f} us mean {w.mean():.2f} (units {uk.sum()})")
c = (ut[..., 3] - ut[..., 2])[uk]
print(f"per unit: converter wait bempty0 -> block 0 done: median {np.median(c):.2f} mean {c.mean():.2f}")
# CTA 0 timeline of first 20 tiles
for i in range(20):
    if ok[0, i]:
        print(f"  tile {i:3d}: mma {tt[0, i, 0]:8.2f}-{tt[0, i, 1]:8.2f}  epi {tt[0, i, 2]:8.2f}-{tt[0, i, 3]:8.2f}")
for u in range(3):
    print(f"  unit {u}: mma waits B0 {ut[0, u, 0]:8.2f} got {ut[0, u, 1]:8.2f} | conv waits bempty0 {ut[0, u, 2]:8.2f} done {ut[0, u, 3]:8.2f}")
