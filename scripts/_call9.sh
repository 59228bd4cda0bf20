EL_DEBUG=1 python paper_2407_20272_b200/build.py --force > gpurun_out/dbg_build.txt 2>&1
timeout 300 python scripts/pipe_gemm_tl.py 256 92 > gpurun_out/pipe_gemm_tl.txt 2>&1
timeout 300 python scripts/pipe_timeline.py 256 92 3 > gpurun_out/pipe_tl_new.txt 2>&1
