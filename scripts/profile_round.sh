#!/bin/bash
# ncu evidence for the round (run under gpurun from the repo root). Outputs in gpurun_out/.
set -x
CFG=${1:-c2}
# 1. launch list of the bench command (eager layer loop: ncu cannot profile kernels inside
#    conditional graphs), 2 timed steps after 3 warm-up
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_${CFG}.csv python bench.py --config $CFG --eager --steps 2 --warmup 3 \
  --no-cpu-baseline > gpurun_out/bench_eager_${CFG}.log 2>&1
# 2. full capture of the dominant kernel (paged attention) and of the GEMMs / LM head
for k in 0 1 4 5; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|attn_kernel" -s 1 -c 1 \
    -o gpurun_out/full_k${k}_${CFG} python scripts/kernel_only.py $k > /dev/null 2>&1
done
ls -la gpurun_out
