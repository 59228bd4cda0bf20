timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest22.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run > gpurun_out/b22_c5.json 2>gpurun_out/b22_c5.err
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-layer-level --no-engine-run > gpurun_out/b22_c2.json 2>gpurun_out/b22_c2.err
