#!/bin/bash
# A/B timing of several builds of the library on the same box:
#   paper_2510_05485_b200/lib_<V>.so  (swapped into libtensorbleu_b200.so in turn)
# usage: AB_VARIANTS="A B C" tools/ab.sh <rounds> [bench args...]   (default variants: A B)
cd "$(dirname "$0")/.."
R=${1:-3}; shift
P=paper_2510_05485_b200
cp $P/libtensorbleu_b200.so /tmp/ab_keep.so
for i in $(seq $R); do
  for v in ${AB_VARIANTS:-A B}; do
    cp $P/lib_$v.so $P/libtensorbleu_b200.so
    out=$(python bench.py --no-cpu-baseline --steps 200 --clock-window 0.3 "$@" | tail -1)
    echo "$v $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,3), 'us/step', round(d['step_flush_l2']['ms_per_step']*1000,3), 'us flushed', round(d['e2e']['value']/1e6,3), 'M e2e')")"
  done
done
cp /tmp/ab_keep.so $P/libtensorbleu_b200.so
