L=paper_2407_20272_b200/libexitlab_b200.so
for rep in 1 2; do
  for v in base pf; do
    cp ab/lib_$v.so $L
    python bench.py --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c5', d['value'], d['ms_per_step'], d['full_layer']['value'])"
  done
done > gpurun_out/ab_pf.txt 2>&1
cp ab/lib_pf.so $L
