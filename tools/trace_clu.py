"""Timeline of the cluster solve (dev tool): python tools/trace_clu.py N"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
tr = torch.zeros(148 * 256 * 16, dtype=torch.int64, device="cuda")
os.environ["PB_CLU_TRACE"] = str(tr.data_ptr())
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
T = tr.cpu().numpy().reshape(148, 256, 16).astype(np.float64)
t0 = T[T > 1000].min()
Tn = np.where(T > 1000, (T - t0) / 1e3, np.nan)
names = ["wait", "data", "x1arr", "x1done", "x2arr", "x2done", "stored", "end"]
r = Tn.reshape(-1, 16)
d = lambda a, b: np.nanmean(r[:, b] - r[:, a])
print(f"mean: wait-data {d(0,1):.2f} sweep1+agg {d(1,2):.2f} x1 {d(2,3):.2f} sweeps2-3 {d(3,4):.2f} x2 {d(4,5):.2f} "
      f"sweep4+store {d(5,6):.2f} release {d(6,7):.2f}")
print(f"detail: vload {d(1,8):.2f} sweep1 {d(8,9):.2f} aggfold {d(9,10):.2f} remote {d(10,2):.2f} | "
      f"fold2(p15) {d(3,11):.2f} sweep2(p15) {d(11,12):.2f} | fold4(p0) {d(5,13):.2f} sweep4(p0) {d(13,14):.2f} zcorr {d(14,15):.2f} store {d(15,6):.2f}")
