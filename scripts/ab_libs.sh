# A/B of library variants in ab/ (same box, interleaved): bench value per config
L=paper_2407_20272_b200/libexitlab_b200.so
cp $L ab/lib_cur.so
for rep in 1 2; do
  for v in "$@"; do
    cp ab/lib_$v.so $L
    for c in ${AB_CONFIGS:-c2 c5}; do
      python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['value'], d['ms_per_step'])"
    done
  done
done
cp ab/lib_cur.so $L
