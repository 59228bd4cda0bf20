#!/bin/bash
# Round-2c evidence (final round-2 code) (under gpurun from the repo root; outputs in gpurun_out/):
#  1. launch list of the default bench command (c5: pipelined kernel, one launch per decode iteration)
#  2. --set full capture of the pipelined kernel at c5 (classifier) and of the persistent kernel at c2
#  3. --set full capture of the per-phase GEMM kernels at c5 and c2 (QKV, W_o, up, down of layer 1):
#     tensor-pipe and DRAM utilisation per projection GEMM
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run > gpurun_out/ncu_bench_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 2 -c 1 \
  -o gpurun_out/full_pipe_c5 python scripts/iter_only.py c5 classifier 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 2 -c 1 \
  -o gpurun_out/full_iter_c2 python scripts/iter_only.py c2 state 3 > /dev/null 2>&1
for c in c5 c2; do
timeout 900 ncu --set full --clock-control none -k regex:gemm_kernel -c 4 \
  -o gpurun_out/full_gemm_$c python scripts/gemm_phase_probe.py $c 1 > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_c5.csv
# summaries on the box (the reports themselves exceed gpurun's 64 MiB copy-back)
python scripts/ncu_summary.py gpurun_out/full_pipe_c5.ncu-rep gpurun_out/iter_traffic_c5.json > gpurun_out/r02c_full_pipe_c5.txt 2>&1
python scripts/ncu_summary.py gpurun_out/full_iter_c2.ncu-rep gpurun_out/iter_traffic_c2.json > gpurun_out/r02c_full_iter_c2.txt 2>&1
for c in c5 c2; do python scripts/ncu_table.py gpurun_out/full_gemm_$c.ncu-rep > gpurun_out/r02c_gemm_$c.txt 2>&1; done
ncu -i gpurun_out/full_pipe_c5.ncu-rep --page source --csv > gpurun_out/r02c_pipe_c5_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/
