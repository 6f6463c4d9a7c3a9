"""One factor + a few pent_solve launches (dev tool for ncu):
python tools/prof_solve.py N [dtype] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dt = sys.argv[2] if len(sys.argv) > 2 else "f64"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
s = synth.SIGMA_STATS
diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=n, n=n, periodic=True, dtype=dt)
x = torch.from_numpy(synth.rhs_uniform(n, n, seed=2)).to("cuda", torch.float64 if dt == "f64" else torch.float32)
for _ in range(reps):
    h.solve(x)
torch.cuda.synchronize()
print("done")
