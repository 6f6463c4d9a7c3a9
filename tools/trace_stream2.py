"""Coupling timeline of the two-phase streaming solve (dev tool): python tools/trace_stream2.py N [lead]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
tr = torch.zeros(148 * 8 * 256 * 8, dtype=torch.int64, device="cuda")
os.environ["PB_STREAM_TRACE"] = str(tr.data_ptr())
os.environ["PB_STREAM"] = "1"
import paper_2101_06550_b200 as pb  # noqa: E402

s = synth.SIGMA_STATS
diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=n, n=n, periodic=True)
x = torch.rand(n * n, dtype=torch.float64, device="cuda")
for _ in range(3):
    tr.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.solve(x)
    e1.record()
    torch.cuda.synchronize()
    print("solve ms", e0.elapsed_time(e1))
T = tr.cpu().numpy().reshape(148, 8, 256, 8).astype(np.float64)
t0 = T[T > 1000].min()
Tn = np.where(T > 1000, (T - t0) / 1e3, np.nan)
# P1 tile completion (sync warp publish) times per CTA: Tn[cta, 5, i, 7]
pub = Tn[:, 5, :, 7]
print("publish times cta0 first 12:", np.round(pub[0, :12], 1))
print("publish times cta63 first 12:", np.round(pub[63, :12], 1))
# per group i: max over CTAs of publish time (kk=0 CTAs: even blockIdx? grid = nrb*K; kk = bid // nrb)
nrb = 64
for kk in (0,):
    ctas = [c for c in range(148) if c // nrb == kk and c < 128]
    mx = np.nanmax(pub[ctas], axis=0)
    mn = np.nanmin(pub[ctas], axis=0)
    print("group i: min/max publish over CTAs (first 12):")
    print("  min", np.round(mn[:12], 1))
    print("  max", np.round(mx[:12], 1))
# scan warp: Tn[cta, 6, j, 0..7]: start poll, count reached, done
sc = Tn[:, 6]
d_poll = sc[:, :, 1] - sc[:, :, 0]
d_scan = sc[:, :, 7] - sc[:, :, 1]
print("scan: mean wait-for-count %.2f us, mean scan %.2f us" % (np.nanmean(d_poll), np.nanmean(d_scan)))
pb_ = Tn[:, 7]
print("producer B: mean flag wait %.2f us" % np.nanmean(pb_[:, :, 1] - pb_[:, :, 0]))
print("P2 flag-ready times cta0 first 12:", np.round(pb_[0, :12, 1], 1))
for cw in range(5):
    r = Tn[:, cw].reshape(-1, 8)
    print(f"consumer {cw}: wait-data {np.nanmean(r[:,1]-r[:,0]):.2f} item {np.nanmean(r[:,7]-r[:,1]):.2f} n={np.sum(~np.isnan(r[:,7]))}")
