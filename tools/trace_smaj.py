"""Dev tool: timeline of the sample-major fused fp16 kernel (TCBF_TRACE, dev build) on the radio
shape -> per-tile MMA / epilogue spans and who waits on whom, summarised over CTAs.
Slots per CTA (gemm_f16_smaj.cu): tile it: [4it] MMA start (TMEM buffer free), [4it+1] MMAs issued,
[4it+2] epilogue warp 2 got the tile, [4it+3] epilogue warp 2 done; [512+4it] ns the MMA issuer
waited for weight stages, [512+4it+1] ns waited for converted data, [512+4it+2] last epilogue warp
done, [512+4it+3] ns the MMA issuer waited for a free TMEM buffer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_03269_b200 as tcbf  # noqa: E402
from paper_2505_03269_b200 import build as _b  # noqa: E402
import synth  # noqa: E402

tcbf.library_path = os.environ.get("TRACE_LIB") or _b.build_tcbf(dev=True)  # TRACE_LIB: a variant build
M, N, K, B = 1024, 1024, int(os.environ.get("TRACE_K", "256")), 256
plan = tcbf.Plan(M, N, K, B, "f16")
wp = plan.pack(tcbf.WEIGHTS, synth.generate_device("phase", 1, 0, B, M, K))
x = synth.generate_device("adc", 1, 1, B, K, N)
out = plan.alloc_output()
for _ in range(int(os.environ.get("TRACE_WARM", "20"))):
    plan.beamform_raw(wp, x, out=out)
torch.cuda.synchronize()
path = "/tmp/smaj_trace.bin"
os.environ["TCBF_TRACE"] = path
plan.beamform_raw(wp, x, out=out)
torch.cuda.synchronize()
del os.environ["TCBF_TRACE"]
t = np.fromfile(path, dtype=np.uint64).reshape(-1, 1024).astype(np.int64)
nc = t.shape[0]
ts = t[:, :512].reshape(nc, 128, 4)
ex = t[:, 512:].reshape(nc, 128, 4)
ok = (ts > 0).all(-1)
t0 = ts[..., 0][ok].min()
tt = np.where(ts > 0, ts - t0, 0) / 1e3
end = tt[..., 3][ok].max()
print(f"kernel span {end:.1f} us, CTAs {nc}, tiles per CTA {ok.sum(1).mean():.1f}")
mma = (tt[..., 1] - tt[..., 0])[ok]
epi = (tt[..., 3] - tt[..., 2])[ok]
epi_last = np.where(ex[..., 2] > 0, (ex[..., 2] - t0) / 1e3 - tt[..., 2], 0)[ok]
print(f"per tile: MMA issue span median {np.median(mma):.2f} us (mean {mma.mean():.2f}); epilogue warp2 "
      f"{np.median(epi):.2f} (mean {epi.mean():.2f}); last epi warp done after {np.median(epi_last):.2f}")
ww = ex[..., 0][ok] / 1e3
xw = ex[..., 1][ok] / 1e3
tw = ex[..., 3][ok] / 1e3
print(f"MMA issuer waits per tile: weights {np.median(ww):.2f} (mean {ww.mean():.2f}) us, data {xw.mean():.2f}, "
      f"TMEM buffer {np.median(tw):.2f} (mean {tw.mean():.2f})")
gap = (tt[..., 2] - tt[..., 1])[ok]
print(f"MMAs issued -> epilogue starts: median {np.median(gap):.2f} us")
st = tt[..., 0]
both = ok[:, 1:] & ok[:, :-1]
d = np.diff(st, axis=1)[both]
print(f"MMA tile start interval: median {np.median(d):.2f} us mean {d.mean():.2f}")
es = tt[..., 2]
d = np.diff(es, axis=1)[both]
print(f"epilogue tile start interval: median {np.median(d):.2f} us mean {d.mean():.2f}")
ee = tt[..., 3]
idle = (es[:, 1:] - ee[:, :-1])[both]
print(f"epilogue warp2 idle between tiles: median {np.median(idle):.2f} us mean {idle.mean():.2f}")
for i in range(12):
    print(f"  CTA0 tile {i:2d}: mma {tt[0, i, 0]:8.2f}-{tt[0, i, 1]:8.2f}  epi {tt[0, i, 2]:8.2f}-{tt[0, i, 3]:8.2f} "
          f" wW {ex[0, i, 0] / 1e3:5.2f} wX {ex[0, i, 1] / 1e3:5.2f} wT {ex[0, i, 3] / 1e3:5.2f}")

