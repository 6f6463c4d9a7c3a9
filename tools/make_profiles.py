"""Copy the judged evidence of a gpu_run.sh call into profiles/ (dev tool):
bench line, launch-list summary, ncu --set full key counters and the
per-launch DRAM traffic bench.py reports as roofline.traffic.
Usage: python tools/make_profiles.py TAG   (reads gpurun_out/)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

tag = sys.argv[1]
out = os.path.join(ROOT, "profiles")
g = os.path.join(ROOT, "gpurun_out")
bench = [l for l in open(os.path.join(g, "bench.log")) if l.startswith("{")]
if bench:
    open(os.path.join(out, f"{tag}_bench.json"), "w").write(bench[-1])
launches = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"),
                           os.path.join(g, "launches.csv")], capture_output=True, text=True).stdout
open(os.path.join(out, f"{tag}_launches.txt"), "w").write(launches)
rows, adi_rows = [], []
for rep in ("prof_band.ncu-rep", "prof_adi.ncu-rep"):
    p = os.path.join(g, rep)
    if os.path.exists(p):
        got = ncu_summary.summarise(p)
        for r in got:
            r["capture"] = "pent_solve cfg2" if rep == "prof_band.ncu-rep" else "one ch_adi_step cfg4"
        rows += got
        if rep == "prof_adi.ncu-rep":
            adi_rows = got
with open(os.path.join(out, f"{tag}_ncu_full.jsonl"), "w") as f:
    for r in rows:
        f.write(json.dumps(r) + "\n")
traffic = {}
for r in rows:
    t = r.get("dram_read", 0) + r.get("dram_write", 0)
    if r["capture"] == "pent_solve cfg2":   # pass 1 + scan + pass 2 of one pent_solve
        traffic["pent_solve_f64"] = traffic.get("pent_solve_f64", 0) + t
    else:                                   # all kernels of one ADI step (pass A + pass B)
        traffic["adi_step_f64"] = traffic.get("adi_step_f64", 0) + t
json.dump(traffic, open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
print(launches)
print(json.dumps(traffic))
