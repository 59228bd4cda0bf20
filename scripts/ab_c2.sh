#!/bin/bash
# same-box A/B at c2 (configs[1], batch 64): engine option sets, two rounds
#   bash scripts/ab_c2.sh "pipe64=0" "pipe64=1 pipe_att_ctas32=84" ...
for r in 1 2; do for set in "$@"; do
  a=""; for kv in $set; do a="$a --opt $kv"; done
  timeout 600 python bench.py --config c2 --no-cpu-baseline $a 2>/dev/null | python -c "
import json, sys
o = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$set', 'run $r', o['value'], 'full', o['full_layer']['value'] if isinstance(o.get('full_layer'), dict) else o.get('full_layer'), 'frac', o['roofline']['frac'], o['roofline'].get('kernel'))"
done; done
