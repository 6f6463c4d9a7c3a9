"""Repeated two-pass solves with a sync after each (dev tool): python tools/tp_repeat.py N M reps"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

n, m, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
nosync = len(sys.argv) > 4 and sys.argv[4] == "nosync"
s = synth.SIGMA_STATS
diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=True)
x = torch.rand(n * m, dtype=torch.float64, device="cuda")
for i in range(reps):
    h.solve(x)
    if not nosync:
        torch.cuda.synchronize()
        print("ok", i, float(x.abs().max()), flush=True)
torch.cuda.synchronize()
print("done", float(x.abs().max()), flush=True)
