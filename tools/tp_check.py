"""Compare the two-pass solve with the cluster path on one shape (dev tool):
python tools/tp_check.py N M [dtype] [periodic 0/1]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
dt = sys.argv[3] if len(sys.argv) > 3 else "f64"
per = (sys.argv[4] != "0") if len(sys.argv) > 4 else True
s = synth.SIGMA_STATS
diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=per, dtype=dt)
x = torch.rand(n * m, dtype=torch.float64 if dt == "f64" else torch.float32, device="cuda")
os.environ["PB_SOLVER"] = "tp"
a = h.solve(x.clone())
torch.cuda.synchronize()
os.environ["PB_SOLVER"] = "tile"
b = h.solve(x.clone())
torch.cuda.synchronize()
print(f"N={n} M={m} {dt} per={per} slab={os.environ.get('PB_TP_SLAB_MB')}: rel diff",
      float((a - b).abs().max() / b.abs().max()), flush=True)
