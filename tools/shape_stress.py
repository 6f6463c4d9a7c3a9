"""Many back-to-back default-path solves on several shapes in one process (dev stress tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
for spec in ["1000:300:f64", "5000:260:f64", "8192:8192:f32", "16384:1024:f64", "2049:40:f32", "777:4096:f64",
             "64:65536:f64", "8192:512:f64"]:
    n, m, dt = spec.split(":")
    n, m = int(n), int(m)
    s = synth.SIGMA_STATS
    diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=True, dtype=dt)
    x = torch.rand(n * m, dtype=torch.float64 if dt == "f64" else torch.float32, device="cuda")
    for _ in range(reps):
        h.solve(x)
    torch.cuda.synchronize()
    print(spec, "ok", float(x.abs().max()), flush=True)
    del h, x
