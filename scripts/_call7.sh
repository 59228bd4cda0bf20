timeout 300 python scripts/attn_grid_probe.py 256 1024 2 3 > gpurun_out/attn_grid2.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run > gpurun_out/b7_c5.json 2>gpurun_out/b7_c5.err
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-layer-level --no-engine-run > gpurun_out/b7_c2.json 2>gpurun_out/b7_c2.err
timeout 300 python bench.py --config c1 --steps 30 --warmup 5 --no-cpu-baseline --no-layer-level --no-engine-run > gpurun_out/b7_c1.json 2>gpurun_out/b7_c1.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest7.log 2>&1
