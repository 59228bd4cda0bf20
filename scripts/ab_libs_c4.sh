#!/bin/bash
# A/B of library variants ab/lib_<v>.so on one box, interleaved: headline c5 + the c4 legs.
#   bash scripts/ab_libs_c4.sh old new
L=paper_2407_20272_b200/libexitlab_b200.so
cp $L ab/lib_cur.so
for rep in 1 2; do
  for v in "$@"; do
    cp ab/lib_$v.so $L
    python bench.py --no-cpu-baseline --no-layer-level --no-engine-run 2>/dev/null | python -c "
import json, sys
o = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'c5', o['value'], {k: (v['value'], v.get('speedup_vs_full_layer')) for k, v in o['c4'].items() if isinstance(v, dict) and 'value' in v})"
  done
done
cp ab/lib_cur.so $L
