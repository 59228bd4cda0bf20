"""Per-launch table of an ncu --set full capture with several launches (one row per launch):
duration, DRAM bytes and throughput, L2 throughput, tensor-pipe utilisation.
    python scripts/ncu_table.py rep.ncu-rep [flops per launch, comma separated]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
flops = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ix = {n: i for i, n in enumerate(h)}
cols = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dram rd"),
        ("dram__bytes_write.sum", "dram wr"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
        ("launch__grid_size", "grid")]
print(" | ".join(c[1] for c in cols) + (" | TFLOP/s" if flops else ""))
for k, r in enumerate(rows[2:]):
    vals = []
    for n, _ in cols:
        v = r[ix[n]] if n in ix else ""
        vals.append(v[:60])
    line = " | ".join(vals)
    if k < len(flops):
        us = float(r[ix["gpu__time_duration.sum"]].replace(",", ""))
        unit = rows[1][ix["gpu__time_duration.sum"]]
        sec = us * (1e-3 if unit == "ns" else 1e-6 if unit == "us" else 1e-3 if unit == "ms" else 1)
        sec = us * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(unit, 1e-6)
        line += f" | {flops[k] / sec / 1e12:.1f}"
    print(line)
print("units:", " | ".join(rows[1][ix[n]] if n in ix else "" for n, _ in cols))
