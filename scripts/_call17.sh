timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest17.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run > gpurun_out/b17_c5.json 2>gpurun_out/b17_c5.err
