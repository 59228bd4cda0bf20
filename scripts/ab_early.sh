#!/bin/bash
# same-box A/B at the driver's default bench (30 steps, early exit ~12 of 24): round-start tree vs
# current library variants and options
L=paper_2407_20272_b200/libexitlab_b200.so
cp $L ab/lib_cur.so
run() {  # label lib opts...
  local lab=$1 lib=$2; shift 2
  cp ab/lib_$lib.so $L
  python bench.py --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run "$@" 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', d['value'], d['ms_per_step'], d['avg_exit_layer'])"
}
for rep in 1 2; do
  (cd ab/orig && python bench.py --no-cpu-baseline --no-c4 --no-layer-level --no-engine-run 2>/dev/null) \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('orig', d['value'], d['ms_per_step'], d['avg_exit_layer'])"
  run now now
  run nolanes nolanes
  run now_att92 now --opt pipe_att_ctas=92
  run now_nows now --opt mega_bm_wstream=0
  run nolanes_att92_nows nolanes --opt pipe_att_ctas=92 --opt mega_bm_wstream=0
done
cp ab/lib_cur.so $L
