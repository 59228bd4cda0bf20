#!/bin/bash
# same-box A/B of the round-start tree (ab/orig, its own bench.py and library) vs the current tree
R=$(pwd)
for rep in 1 2; do
  (cd ab/orig && python bench.py --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null) \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('orig', d['value'], d['ms_per_step'], d['avg_exit_layer'], d['exit_layers'])"
  python bench.py --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('now ', d['value'], d['ms_per_step'], d['avg_exit_layer'], d['exit_layers'])"
done
