"""Key metrics of one kernel in an ncu --set full report -> JSON (what profiles/ summarizes).

usage: python scripts/ncu_summary.py <report.ncu-rep> [kernel-substring]
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_cycles_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
}
out = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if kern and kern not in d.get("Kernel Name", ""):
        continue
    e = {"kernel": d.get("Kernel Name")}
    for k, nm in want.items():
        if k in d and d[k] not in ("", "n/a"):
            try:
                e[nm] = float(d[k].replace(",", ""))
            except ValueError:
                e[nm] = d[k]
            e[nm + "_unit"] = units[hdr.index(k)]
    stalls = {k.split("__")[-1].replace(".pct", ""): float(d[k]) for k in hdr
              if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio") and d.get(k)}
    if not stalls:
        stalls = {k: float(d[k]) for k in hdr if "warps_issue_stalled_" in k and k.endswith("_per_warp_active.pct")
                  and d.get(k)}
    e["stalls"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:10])
    out.append(e)
print(json.dumps(out, indent=1))
