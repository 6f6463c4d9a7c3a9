"""pent_solve on an N x M interleaved batch (dev tool for ncu): python tools/prof_solve2.py N M [dtype] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
dt = sys.argv[3] if len(sys.argv) > 3 else "f64"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
s = synth.SIGMA_STATS
diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=True, dtype=dt)
x = torch.rand(n * m, dtype=torch.float64 if dt == "f64" else torch.float32, device="cuda")
for _ in range(reps):
    h.solve(x)
torch.cuda.synchronize()
print("done")
