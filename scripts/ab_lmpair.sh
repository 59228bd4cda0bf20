#!/bin/bash
# same-box A/B of the softmax-check LM pair units (lm_pair 0 / 1 / 2): the c4 legs
for r in 1 2; do for k in ${LMP_VALUES:-0 1 2}; do
  timeout 600 python bench.py --no-cpu-baseline --no-layer-level --no-engine-run --opt lm_pair=$k > gpurun_out/lmp_${k}_$r.json 2>/dev/null
  python - "$k" "$r" <<'PY'
import json, sys
o = json.loads(open(f"gpurun_out/lmp_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
c4 = o.get("c4", {})
print("lm_pair", sys.argv[1], "run", sys.argv[2], "c5", o["value"],
      {k: (v["value"], v.get("speedup_vs_full_layer"), v.get("layers_per_token")) for k, v in c4.items() if isinstance(v, dict) and "value" in v})
PY
done; done
