# phase timelines under option variants (c2, state technique)
for o in '{}' '{"mega_down_splits":12}' '{"mega_down_splits":16}' '{"mega_down_splits":24}' '{"mega_fill_splits":2}' '{"mega_fill_splits":6}'; do echo "== $o"; python scripts/mega_phases.py ${1:-c2} state "$o" 2>&1 | grep -E "^(qkv|attn|wo|up|down|tail)|timed"; done
