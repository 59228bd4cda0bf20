# option sweep on one box: full-depth iteration time (mega_phases "timed") per option set
cfg=$1; tech=$2; shift 2
for o in "$@"; do
  echo "== $o"; python scripts/mega_phases.py $cfg $tech "$o" 2>&1 | grep -E "^(qkv|attn|wo|up|down|tail)|timed|^down \(|arrival"
done
