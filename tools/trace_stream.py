"""Per-item timeline of the streaming solve (dev tool): python tools/trace_stream.py N [M]
Stamps (us): 0 wait-full, 1 data, 2 fwd sweep+scan, 3 flag (P2), 4 publish (P1) / pre-store (P2),
5 atomic (P1), 6 group scan done, 7 end."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
m = int(sys.argv[2]) if len(sys.argv) > 2 else n
TEAMS = 8
tr = torch.zeros(148 * TEAMS * 256 * 8, dtype=torch.int64, device="cuda")
os.environ["PB_STREAM_TRACE"] = str(tr.data_ptr())
import paper_2101_06550_b200 as pb  # noqa: E402

s = synth.SIGMA_STATS
diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=True)
x = torch.rand(n * m, dtype=torch.float64, device="cuda")
for _ in range(3):
    tr.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.solve(x)
    e1.record()
    torch.cuda.synchronize()
    print("solve ms", e0.elapsed_time(e1), "GB/s", 16 * n * m / e0.elapsed_time(e1) / 1e6)
T = tr.cpu().numpy().reshape(148, TEAMS, 256, 8).astype(np.float64)
t0 = T[T > 1000].min()
Tn = np.where(T > 1000, (T - t0) / 1e3, np.nan)
for cta in (0, 37, 147):
    for team in range(TEAMS):
        print(f"cta {cta} team {team}")
        for r in Tn[cta, team, 10:16]:
            print("   " + " ".join("%8.2f" % v for v in r))
for team in range(TEAMS):
    r = Tn[:, team].reshape(-1, 8)
    d = lambda a, b: np.nanmean(r[:, b] - r[:, a])
    print(f"team {team}: wait-data {d(0,1):.2f}  sweep1+scan {d(1,2):.2f}  ->flag {d(2,3):.2f}  ->4 {d(2,4):.2f} "
          f"atomic {d(4,5):.2f}  scan {d(5,6):.2f}  item {d(1,7):.2f}  n={np.sum(~np.isnan(r[:,7]))}")
