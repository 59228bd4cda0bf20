#!/bin/bash
# same-box A/B of library variants at the driver's default bench length (30 steps, 5 warm-up)
L=paper_2407_20272_b200/libexitlab_b200.so
cp $L ab/lib_cur.so
for rep in 1 2; do
  for v in "$@"; do
    cp ab/lib_$v.so $L
    python bench.py --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['avg_exit_layer'], d['exit_layers'])"
  done
done
cp ab/lib_cur.so $L
