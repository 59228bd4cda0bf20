set -x
timeout 300 python scripts/attn_grid_probe.py 256 1024 2 3 > gpurun_out/attn_grid.txt 2>&1
timeout 300 python bench.py --config c1 --steps 30 --warmup 5 --no-cpu-baseline --no-layer-level --no-engine-run > gpurun_out/c1_auto.json 2>gpurun_out/c1_auto.err
timeout 300 python bench.py --config c1 --mega --steps 30 --warmup 5 --no-cpu-baseline --no-layer-level --no-engine-run > gpurun_out/c1_mega.json 2>gpurun_out/c1_mega.err
EL_DEBUG=1 python paper_2407_20272_b200/build.py --force > gpurun_out/dbg_build.txt 2>&1
for ga in 92 100 108; do timeout 300 python scripts/pipe_timeline.py 256 $ga 24 > gpurun_out/pipe_tl_$ga.txt 2>&1; done
