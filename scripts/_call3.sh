timeout 600 ./scripts/ingest_probe > gpurun_out/ingest.txt 2>&1
EL_DEBUG=1 python paper_2407_20272_b200/build.py --force > gpurun_out/dbg_build.txt 2>&1
ATTN_DBG=1 timeout 300 python scripts/attn_grid_probe.py 256 1024 2 3 > gpurun_out/attn_grid_nomath.txt 2>&1
