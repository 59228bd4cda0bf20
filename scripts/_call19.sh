for i in 1 2; do
for ws in 1 0; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run --opt mega_bm_wstream=$ws > gpurun_out/b19_ws$ws.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b19_ws$ws.json')); print('ws $ws', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done; done > gpurun_out/b19.txt
