"""Tile-configuration sweep of pent_solve (dev tool, not part of the product):
for each N (batch = N), dtype and PB_TILE_CFG, time K back-to-back in-place
solves with CUDA events and print GB/s of algorithmic traffic (2*sizeof(T)
per unknown).  Usage: python tools/sweep.py [--ns 1024,8192] [--k 30]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(n, dtype, cfg, k, periodic, layout):
    import torch
    import synth
    import paper_2101_06550_b200 as pb
    if cfg is not None:
        os.environ["PB_TILE_CFG"] = str(cfg)
    else:
        os.environ.pop("PB_TILE_CFG", None)
    s = synth.SIGMA_STATS
    diags = synth.const_penta(n, s, -4 * s, 1 + 6 * s, -4 * s, s)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    h = pb.pent_factor(*[torch.from_numpy(v).cuda() for v in diags], batch=n, n=n, periodic=periodic, dtype=dtype)
    x = torch.from_numpy(synth.rhs_uniform(n, n, seed=2)).to("cuda", tdt)
    for _ in range(3):
        h.solve(x, layout=layout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        h.solve(x, layout=layout)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    es = 8 if dtype == "f64" else 4
    return {"n": n, "dtype": dtype, "cfg": cfg, "periodic": periodic, "layout": layout, "us": round(ms * 1e3, 2),
            "GBs": round(2 * es * n * n / (ms * 1e-3) / 1e9, 1), "Gunk_s": round(n * n / (ms * 1e-3) / 1e9, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="256,512,1024,2048,4096,8192")
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--cfgs", default="auto,0,1,2,3,4")
    ap.add_argument("--layouts", default="interleaved")
    ap.add_argument("--k", type=int, default=30)
    ap.add_argument("--child", default=None)
    a = ap.parse_args()
    if a.child:
        n, dtype, cfg, per, layout = a.child.split(":")
        r = one(int(n), dtype, None if cfg == "auto" else int(cfg), a.k, per == "1", layout)
        print(json.dumps(r), flush=True)
        return
    for layout in a.layouts.split(","):
        for dtype in a.dtypes.split(","):
            for n in map(int, a.ns.split(",")):
                for cfg in a.cfgs.split(","):
                    # fresh process per config: PB_TILE_CFG is read at factor time
                    p = subprocess.run([sys.executable, __file__, "--k", str(a.k), "--child",
                                        f"{n}:{dtype}:{cfg}:1:{layout}"], capture_output=True, text=True, timeout=300)
                    out = p.stdout.strip().splitlines()
                    print(out[-1] if out and p.returncode == 0 else json.dumps(
                        {"n": n, "dtype": dtype, "cfg": cfg, "error": p.stderr.strip()[-300:]}), flush=True)


if __name__ == "__main__":
    main()
