EL_DEBUG=1 python paper_2407_20272_b200/build.py --force > gpurun_out/dbg_build.txt 2>&1
timeout 300 python scripts/pipe_tail.py > gpurun_out/pipe_tail.txt 2>&1
