#!/bin/bash
# Round-2 evidence (run under gpurun from the repo root; outputs in gpurun_out/):
#  1. launch list of the default bench command (c5: the pipelined iteration kernel, one launch per
#     decode iteration; the e2e and full-layer legs add theirs)
#  2. one --set full capture of the pipelined kernel at c5 (classifier) and of the persistent
#     kernel at c2 (state), bench-shaped (scripts/iter_only.py)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c4 --no-layer-level > gpurun_out/ncu_bench_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 2 -c 1 \
  -o gpurun_out/full_pipe_c5 python scripts/iter_only.py c5 classifier 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 2 -c 1 \
  -o gpurun_out/full_iter_c2 python scripts/iter_only.py c2 state 3 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_c5.csv
