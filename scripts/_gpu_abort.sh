L=paper_2407_20272_b200/libexitlab_b200.so
for rep in 1 2; do
  for v in abort2 np3; do
    cp ab/lib_$v.so $L
    for c in c5; do
    python bench.py --config $c --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['value'], d['ms_per_step'], d['full_layer']['value'])"
    done
  done
done > gpurun_out/ab_abort.txt 2>&1
cp ab/lib_abort2.so $L
