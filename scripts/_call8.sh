EL_DEBUG=1 python paper_2407_20272_b200/build.py --force > gpurun_out/dbg_build.txt 2>&1
for a in "37 2" "37 3" "148 2"; do timeout 120 python scripts/attn_tl2.py 256 1024 $a; done > gpurun_out/attn_tl2.txt 2>&1
ATTN_DBG=1 timeout 300 python scripts/attn_grid_probe.py 256 1024 2 3 > gpurun_out/attn_grid_nomath2.txt 2>&1
