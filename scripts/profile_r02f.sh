#!/bin/bash
# Round-2f evidence (final round-2 code) (under gpurun from the repo root; outputs in gpurun_out/):
#  1. bench lines: c5 (default, all legs), c3, c2, c1, and the reference arm
#  2. launch list of the default bench command (c5: one pipe_kernel launch per decode iteration)
#  3. --set full capture of the pipelined kernel at c5 (classifier) and of the pipelined kernel at
#     c4 softmax (LM check on the GEMM CTAs, transposed pair units), summaries written on the box
python bench.py > gpurun_out/r02f_bench_c5.json 2> gpurun_out/r02f_bench_c5.err
for c in c3 c2 c1; do python bench.py --config $c > gpurun_out/r02f_bench_$c.json 2> gpurun_out/r02f_bench_$c.err; done
python bench.py --impl reference > gpurun_out/r02f_ref.json 2> gpurun_out/r02f_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02f_launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run > gpurun_out/ncu_bench_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 2 -c 1 \
  -o gpurun_out/full_pipe_c5 python scripts/iter_only.py c5 classifier 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 2 -c 1 \
  -o gpurun_out/full_pipe_c4m python scripts/iter_only.py c4m softmax 3 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/full_pipe_c5.ncu-rep gpurun_out/iter_traffic_c5.json > gpurun_out/r02f_full_pipe_c5.txt 2>&1
python scripts/ncu_summary.py gpurun_out/full_pipe_c4m.ncu-rep gpurun_out/iter_traffic_c4m.json > gpurun_out/r02f_full_pipe_c4m.txt 2>&1
python scripts/launches.py gpurun_out/r02f_launches_c5.csv > gpurun_out/r02f_launches_c5_summary.txt 2>&1
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/
