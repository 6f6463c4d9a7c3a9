"""Key counters of every kernel in an ncu --set full report (dev tool):
duration, DRAM bytes read/written (per launch), DRAM throughput %, achieved
occupancy, registers, L2 hit rate, shared-memory bank conflicts.
Usage: python tools/ncu_summary.py report.ncu-rep [--json traffic_key]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__cluster_dim_x": "cluster",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}


def summarise(path):
    """path: an .ncu-rep, or the `--page raw --csv` export of one (*.raw.csv)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0][:90]}
        for k, name in KEYS.items():
            if k in h:
                i = h.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * UNIT.get(units[i], 1)
        res.append(d)
    return res


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    for d in res:
        print(json.dumps(d))
