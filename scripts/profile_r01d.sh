#!/bin/bash
# Round-1d evidence (run under gpurun from the repo root; outputs in gpurun_out/):
#  1. launch list of the default bench command (persistent kernel: one launch per decode iteration)
#  2. one --set full capture of the persistent kernel at c2 (state) and c5 (classifier), bench-shaped
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:iter_kernel --log-file gpurun_out/launches_c2.csv \
  python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 2 -c 1 \
  -o gpurun_out/full_iter_c2 python scripts/iter_only.py c2 state 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 2 -c 1 \
  -o gpurun_out/full_iter_c5 python scripts/iter_only.py c5 classifier 3 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_c2.csv
