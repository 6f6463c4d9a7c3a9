"""pent_solve throughput on arbitrary (N, M) shapes (dev tool): python tools/sweep_shapes.py N:M[:dtype] ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_06550_b200 as pb  # noqa: E402

for spec in sys.argv[1:]:
    parts = spec.split(":")
    n, m = int(parts[0]), int(parts[1])
    dt = parts[2] if len(parts) > 2 else "f64"
    per = (parts[3] != "np") if len(parts) > 3 else True
    s = synth.SIGMA_STATS
    diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=m, n=n, periodic=per, dtype=dt)
    x = torch.rand(n * m, dtype=torch.float64 if dt == "f64" else torch.float32, device="cuda")
    for _ in range(3):
        h.solve(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 10
    e0.record()
    for _ in range(k):
        h.solve(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    es = 8 if dt == "f64" else 4
    print(f"N={n} M={m} {dt} periodic={per}: {ms*1e3:9.1f} us  {2*es*n*m/(ms*1e-3)/1e9:8.1f} GB/s", flush=True)
    del x, h
    torch.cuda.empty_cache()
