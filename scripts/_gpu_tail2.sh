timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest45.log 2>&1
for rep in 1 2; do
  (cd ab/orig && python bench.py --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('orig', d['value'], d['ms_per_step'], d['full_layer']['value'])"
  python bench.py --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new ', d['value'], d['ms_per_step'], d['full_layer']['value'])"
done > gpurun_out/ab_tail.txt 2>&1
EL_DEBUG=1 python paper_2407_20272_b200/build.py --force > gpurun_out/dbg_build.txt 2>&1
timeout 300 python scripts/pipe_tail.py > gpurun_out/pipe_tail.txt 2>&1
