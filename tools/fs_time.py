"""Timing + sampled oracle check of pent_solve at several (n, m) shapes (dev tool):
python tools/fs_time.py [f64|f32] n:m ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] in ("f64", "f32") else "f64"
shapes = [a for a in sys.argv[1:] if ":" in a] or ["8192:8192", "4096:4096", "2048:2048", "1024:1024", "512:262144"]
tdt = torch.float64 if dt == "f64" else torch.float32
es = 8 if dt == "f64" else 4
for sh in shapes:
    n, m = (int(v) for v in sh.split(":"))
    s = synth.SIGMA_STATS
    diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=True, dtype=dt)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    f = (torch.rand(n * m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).to(tdt)
    x = f.clone()
    h.solve(x)
    torch.cuda.synchronize()
    F = f.double().view(n, m)
    X = x.double().view(n, m)
    err = 0.0
    for sy in sorted({0, 1, m // 2, m - 1}):
        ref = oracle.penta_batch_solve(*diags, F[:, sy].cpu().numpy().copy(), n=n, m=1, periodic=True)
        err = max(err, float(np.max(np.abs(X[:, sy].cpu().numpy() - ref)) / np.max(np.abs(ref))))
    for _ in range(5):
        h.solve(x)
    reps = max(10, min(200, int(4e9 / (n * m * es))))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        h.solve(x)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    gbs = 2 * es * n * m / (us * 1e-6) / 1e9
    print(f"{dt} n={n} m={m}: {us:9.2f} us/solve  {gbs:7.1f} GB/s alg  ({gbs / 6539.9:.3f} of HBM)  sampled relerr {err:.2e}",
          flush=True)
    h.close()
    del x, f
    torch.cuda.empty_cache()
