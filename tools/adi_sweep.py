"""ch_adi_step timing at cfg4 (512 sims x 512^2 fp64) for the current env (dev tool)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

n, sims = 512, int(sys.argv[1]) if len(sys.argv) > 1 else 512
L = 4 * math.pi
dt = synth.ch_dt(n, L)
c0 = torch.from_numpy(synth.ch_ic_random(sims, n, seed=1)).cuda()
st = pb.CHState(c0)
pb.ch_adi_step(st, dt, D=1.0, gamma=0.01, L=L, nsteps=3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pb.ch_adi_step(st, dt, D=1.0, gamma=0.01, L=L, nsteps=20)
e1.record()
torch.cuda.synchronize()
print(f"ADI cfg4: "
      f"{e0.elapsed_time(e1) / 20:.3f} ms/step", flush=True)
