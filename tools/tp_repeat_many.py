"""Repeated pent_solve_many at the ADI shape (dev stress tool):
python tools/tp_repeat_many.py N M COUNT REPS"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

n, m, cnt, reps = (int(a) for a in sys.argv[1:5])
s = synth.SIGMA_STATS
diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=True)
x = torch.rand(cnt * n * m, dtype=torch.float64, device="cuda")
for i in range(reps):
    h.solve_many(x, cnt, n * m)
torch.cuda.synchronize()
print("done", float(x.abs().max()), flush=True)
