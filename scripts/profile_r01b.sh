#!/bin/bash
# ncu evidence for round 1 (run under gpurun from the repo root). Outputs in gpurun_out/.
#  1. launch lists (per-launch device time + DRAM bytes) of bench.py at c2 (per-phase kernels,
#     eager layer loop: ncu cannot profile kernels inside conditional graphs) and c5 / c2t5
#     (persistent kernel: one launch per decode iteration)
#  2. one --set full capture of the dominant kernel of each: attn_kernel (c2), iter_kernel (c5, c2t5)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --config c2 --eager --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_c2.log 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:iter_kernel --log-file gpurun_out/launches_c5.csv \
  python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_c5.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 1 -c 1 \
  -o gpurun_out/full_attn_c2 python scripts/kernel_only.py 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 2 -c 1 \
  -o gpurun_out/full_iter_c5 python scripts/iter_only.py c5 classifier 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 2 -c 1 \
  -o gpurun_out/full_iter_c2t5 python scripts/iter_only.py c2t5 state 3 > /dev/null 2>&1
ls -la gpurun_out
