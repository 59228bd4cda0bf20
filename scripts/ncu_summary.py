"""Key metrics of an ncu --set full capture (one launch) -> text summary; optional traffic JSON.
    python scripts/ncu_summary.py rep.ncu-rep [traffic.json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
get = {n: (v[i], units[i]) for i, n in enumerate(h)}
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tma.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "smsp__average_warp_latency_per_inst_issued.ratio"]
out = []
for n in want:
    if n in get:
        out.append(f"{n:70s} {get[n][0]} {get[n][1]}")
stalls = sorted(((float(get[n][0] or 0), n) for n in get
                 if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")),
                reverse=True)[:8]
out.append("top stall reasons (warps per issue-active cycle):")
for val, n in stalls:
    out.append(f"   {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {val:.3f}")
print("\n".join(out))
if len(sys.argv) > 2:
    def num(n):
        x, u = get[n]
        x = float(x.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    t = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    with open(sys.argv[2], "w") as f:
        json.dump({"source": rep.split("/")[-1], "dram_bytes_per_launch": t,
                   "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
                   "duration_us_under_ncu": float(get["gpu__time_duration.sum"][0].replace(",", "")) *
                   {"ns": 1e-3, "us": 1.0, "ms": 1e3}[get["gpu__time_duration.sum"][1]]}, f, indent=1)
