"""Debug helper: streaming-conversion kernel vs pack + beamform, repeated, with the mismatch pattern."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03269_b200 as tcbf
import synth
os.environ["TCBF_CONV_SPLITS"] = "1"
os.environ["TCBF_FORCE_STREAM_CONV"] = "1"
SH = [(32, 256, 1024, 80, "interleaved"), (32, 256, 1000, 80, "interleaved"), (128, 256, 1024, 80, "interleaved"),
      (32, 8192, 1024, 1, "interleaved"), (32, 256, 256, 4, "interleaved")]
for (M, N, K, B, layout) in SH:
    w = synth.generate("phase", 17, 0, B, M, K)
    x = synth.generate("adc", 17, 1, B, K, N)
    conv = synth.to_interleaved if layout == "interleaved" else synth.to_planar
    plan = tcbf.Plan(M, N, K, B, "f16")
    wp = plan.pack(tcbf.WEIGHTS, torch.from_numpy(conv(w)).cuda(), layout)
    xd = torch.from_numpy(conv(x)).cuda()
    y_ref = plan.beamform(wp, plan.pack(tcbf.DATA, xd, layout))
    out = torch.empty_like(y_ref)
    bad = 0
    for r in range(8):
        out.fill_(float("nan"))
        plan.beamform_raw(wp, xd, layout, out=out)
        torch.cuda.synchronize()
        d = (out - y_ref).abs()
        m = ~(d == 0)
        if m.any():
            bad += 1
            idx = torch.nonzero(m)
            nan = torch.isnan(out).sum().item()
            print(f"  run {r}: n_diff {idx.shape[0]} nan {nan} max {d[~torch.isnan(d)].max().item() if (~torch.isnan(d)).any() else 0:.3g} "
                  f"batches {sorted(set(idx[:, 0].tolist()))[:8]} planes {sorted(set(idx[:, 1].tolist()))} "
                  f"rows {sorted(set(idx[:, 2].tolist()))[:10]} cols {sorted(set(idx[:, 3].tolist()))[:40]}", flush=True)
    print(M, N, K, B, layout, "bad runs", bad, "of 8", flush=True)
