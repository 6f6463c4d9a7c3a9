"""stencil_apply on one 8192^2 fp64 grid with the 13-point biharmonic window
(5x5, periodic), 3 launches: the ncu capture target of stencil_kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_06550_b200 as pb  # noqa: E402

n = 8192
g = torch.rand((1, n, n), dtype=torch.float64, device="cuda")
o = torch.empty_like(g)
w = np.zeros((5, 5))
w[2, :] += [1, -4, 6, -4, 1]
w[:, 2] += [1, -4, 6, -4, 1]
w[1:4, 1:4] += 2 * np.array([[1, -2, 1], [-2, 4, -2], [1, -2, 1]])
for _ in range(3):
    pb.stencil_apply(g, o, w.reshape(-1), left=2, right=2, top=2, bottom=2, periodic=True)
torch.cuda.synchronize()
print("done")
