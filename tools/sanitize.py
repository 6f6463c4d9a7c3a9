"""Small invocations of every kernel family for compute-sanitizer (dev tool):
compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize.py"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

s = synth.SIGMA_STATS
for (n, m, dt) in [(1024, 96, "f64"), (700, 40, "f32"), (256, 64, "f64"), (2048, 32, "f64")]:
    for per in (True, False):
        diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
        h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=per, dtype=dt)
        x = torch.from_numpy(synth.rhs_uniform(n, m, seed=1)).cuda().to(torch.float64 if dt == "f64" else torch.float32)
        h.solve(x)
        h.solve(x, layout="contiguous")
        h.close()
c0 = torch.from_numpy(synth.ch_ic_random(2, 64, seed=3)).cuda()
st = pb.CHState(c0)
pb.ch_adi_step(st, 0.001, L=2 * math.pi, nsteps=2)
c1 = torch.from_numpy(np.random.default_rng(0).uniform(-0.1, 0.1, (256, 64))).cuda()
s1 = pb.CH1DState(c1)
pb.ch1d_step(s1, 0.001, L=2 * math.pi, nsteps=2)
g = torch.randn(2, 40, 70, dtype=torch.float64, device="cuda")
o = torch.zeros_like(g)
pb.stencil_apply(g, o, np.ones(9), left=1, right=1, top=1, bottom=1, periodic=True)
torch.cuda.synchronize()
print("sanitize run done")
