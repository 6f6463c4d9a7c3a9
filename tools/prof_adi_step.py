"""One cfg4 ADI step after warm-up (the ncu capture target of the ADI kernels):
python tools/prof_adi_step.py [sims]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

n, sims = 512, int(sys.argv[1]) if len(sys.argv) > 1 else 512
L = n * synth.DX_STATS
dt = synth.ch_dt(n, L)
g = torch.Generator(device="cuda")
g.manual_seed(4)
c0 = torch.rand((sims, n, n), dtype=torch.float64, device="cuda", generator=g) * 0.2 - 0.1
st = pb.CHState(c0)
pb.ch_adi_step(st, dt, D=1.0, gamma=0.01, L=L, nsteps=3)
torch.cuda.synchronize()
pb.ch_adi_step(st, dt, D=1.0, gamma=0.01, L=L, nsteps=1)
torch.cuda.synchronize()
print("done")
