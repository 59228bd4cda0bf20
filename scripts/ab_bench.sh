#!/bin/bash
# A/B of library variants ab/lib_<v>.so on one box, interleaved: bench value per config.
#   bash scripts/ab_bench.sh v1 v2 ...   (AB_CONFIGS="c5 c2" by default)
L=paper_2407_20272_b200/libexitlab_b200.so
cp $L ab/lib_cur.so
for rep in 1 2; do
  for v in "$@"; do
    cp ab/lib_$v.so $L
    for c in ${AB_CONFIGS:-c5 c2}; do
      python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['value'], d['ms_per_step'])"
    done
  done
done
cp ab/lib_cur.so $L
