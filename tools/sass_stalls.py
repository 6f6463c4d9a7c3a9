"""Top stall sites of an ncu report's SASS page (dev tool):
python tools/sass_stalls.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
print("total samples", tot)
keys = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
idx = {k: h.index(k) for k in keys}
agg = {}
for r in data:
    for k, i in idx.items():
        if r[i].isdigit():
            agg[k] = agg.get(k, 0) + int(r[i])
print({k: round(v / tot, 3) for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v / tot > 0.01})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(data, key=lambda r: -int(r[iS]) if r[iS].isdigit() else 0)[:n]:
    print(r[0][-5:], r[iS], r[1][:70], {k[6:]: r[i] for k, i in idx.items() if r[i] not in ("0", "")})
