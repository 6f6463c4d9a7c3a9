"""A few steps of the thesis's 1D CH batch (2^20 x 256, fp64): ncu capture target."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

n, m, L = 256, 1 << 20, 2 * math.pi
dt = synth.ch_dt(n, L)
c0 = torch.empty((n, m), dtype=torch.float64, device="cuda").uniform_(-0.1, 0.1)
st = pb.CH1DState(c0)
pb.ch1d_step(st, dt, gamma=0.01, L=L, nsteps=5)
torch.cuda.synchronize()
print("done")
