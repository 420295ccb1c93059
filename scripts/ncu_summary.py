"""Summarise an ncu --set full report (raw page) for the SpMV kernel into JSON."""
import csv, json, subprocess, sys
rep, out_key = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
get = lambda k: (vals[hdr.index(k)], units[hdr.index(k)]) if k in hdr else (None, None)
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "smsp__warps_eligible.avg.per_cycle_active", "launch__grid_size", "launch__block_size"]
d = {}
for k in keys:
    v, u = get(k)
    if v is not None:
        d[k] = v + ("" if not u else " " + u)
stalls = {}
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
        try:
            stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(vals[i]))
        except ValueError:
            pass
tot = sum(stalls.values()) or 1
d["stall_samples_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda t: -t[1])[:8]}
rd = float(vals[hdr.index("dram__bytes_read.sum")]) if "dram__bytes_read.sum" in hdr else 0
print(json.dumps({out_key: d}, indent=1))
