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
lname = f"{tag}_launches.csv" if os.path.exists(os.path.join(g, f"{tag}_launches.csv")) else "launches.csv"
if os.path.exists(os.path.join(g, lname)):
    launches = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"),
                               os.path.join(g, lname)], capture_output=True, text=True).stdout
    open(os.path.join(out, f"{tag}_launches.txt"), "w").write(launches)
    print(launches)
# (capture file, what, traffic key, launches per unit of work: the per-launch
# traffic of a multi-launch unit is the sum over its launches; captures holding
# several units are averaged)
captures = {f"{tag}_solve.raw.csv": ("pent_solve cfg2 N=M=8192 fp64 (P1, scan, P2)", "pent_solve_f64", 3),
            f"{tag}_solve32.raw.csv": ("pent_solve cfg2 N=M=8192 fp32 (P1, scan, P2)", "pent_solve_f32", 3),
            f"{tag}_adi.raw.csv": ("one ch_adi_step cfg4 fp64 (rhs, x-sweep P1/scan/P2, y-sweep, combine)", "adi_step_f64", 6),
            f"{tag}_ch1d.raw.csv": ("one ch1d_step 2^20 x 256 fp64", "ch1d_f64", 1),
            f"{tag}_stencil.raw.csv": ("stencil_apply 5x5 periodic on 8192^2 fp64", "stencil_f64", 1)}
rows, traffic = [], {}
for rep, (what, key, per) in captures.items():
    p = os.path.join(g, rep)
    if not os.path.exists(p):
        continue
    rs = ncu_summary.summarise(p)
    tot = 0.0
    for r in rs:
        r["capture"] = what
        rows.append(r)
        tot += r.get("dram_read", 0) + r.get("dram_write", 0)
    units = max(1, len(rs) // per)
    traffic[key] = tot / units
with open(os.path.join(out, f"{tag}_ncu_full.jsonl"), "w") as f:
    for r in rows:
        f.write(json.dumps(r) + "\n")
json.dump(traffic, open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(traffic))
