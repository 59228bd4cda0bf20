#!/bin/bash
# same-box A/B of one engine option over the bench (headline c5 + the c4 legs), two rounds:
#   OPT=lm_tail VALUES="0 1" bash scripts/ab_opt.sh
for r in 1 2; do for k in $VALUES; do
  timeout 600 python bench.py --no-cpu-baseline --no-layer-level --no-engine-run --opt $OPT=$k > gpurun_out/ab_${OPT}_${k}_$r.json 2>/dev/null
  python - "$OPT" "$k" "$r" <<'PY'
import json, sys
o = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}_{sys.argv[3]}.json").read().strip().splitlines()[-1])
c4 = o.get("c4", {})
print(sys.argv[1], sys.argv[2], "run", sys.argv[3], "c5", o["value"], "frac", o["roofline"]["frac"],
      {k: (v["value"], v.get("speedup_vs_full_layer")) for k, v in c4.items() if isinstance(v, dict) and "value" in v})
PY
done; done
