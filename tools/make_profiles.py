"""Copy the judged evidence of a tools/jobs/profile.sh call into profiles/ (dev
tool): the bench line, the launch list summary, the key ncu --set full counters
of every captured kernel and the per-launch DRAM traffic bench.py reports as
roofline.traffic.   Usage: python tools/make_profiles.py TAG   (reads gpurun_out/)"""
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
bench = [l for l in open(os.path.join(g, "bench.log")) if l.startswith("{")] if os.path.exists(
    os.path.join(g, "bench.log")) else []
if bench:
    open(os.path.join(out, f"{tag}_bench.json"), "w").write(bench[-1])
if os.path.exists(os.path.join(g, "launches.csv")):
    launches = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"),
                               os.path.join(g, "launches.csv")], capture_output=True, text=True).stdout
    open(os.path.join(out, f"{tag}_launches.txt"), "w").write(launches)
    print(launches)
captures = {"prof_band.ncu-rep": ("pent_solve cfg2 N=M=8192 fp64", "pent_solve_f64"),
            "prof_band32.ncu-rep": ("pent_solve cfg2 N=M=8192 fp32", "pent_solve_f32"),
            "prof_adi.ncu-rep": ("one ch_adi_step cfg4 fp64", "adi_step_f64"),
            "prof_ch1d.ncu-rep": ("one ch1d_step 2^20 x 256 fp64", "ch1d_f64"),
            "prof_stencil.ncu-rep": ("stencil_apply 5x5 on 64 x 1024^2 fp64", "stencil_f64")}
rows, traffic = [], {}
for rep, (what, key) in captures.items():
    p = os.path.join(g, rep)
    if not os.path.exists(p):
        continue
    for r in ncu_summary.summarise(p):
        r["capture"] = what
        rows.append(r)
        traffic[key] = traffic.get(key, 0) + r.get("dram_read", 0) + r.get("dram_write", 0)
with open(os.path.join(out, f"{tag}_ncu_full.jsonl"), "w") as f:
    for r in rows:
        f.write(json.dumps(r) + "\n")
json.dump(traffic, open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(traffic))
