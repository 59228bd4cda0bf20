timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest14.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run > gpurun_out/b14_c5.json 2>gpurun_out/b14_c5.err
EL_DEBUG=1 python paper_2407_20272_b200/build.py --force > gpurun_out/dbg_build.txt 2>&1
timeout 300 python scripts/pipe_timeline.py 256 100 3 > gpurun_out/pipe_tl14.txt 2>&1
timeout 300 python scripts/pipe_gemm_tl.py 256 100 > gpurun_out/pipe_gemm_tl14.txt 2>&1
