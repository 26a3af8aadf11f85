#!/bin/bash
# A/B of liblrc.so builds: bash tools/unroll_sweep.sh u2 p2 ... (var_<v>.so in _lib/)
# Decode-only bench at B=1 and B=8 per variant (phase times included).
L=paper_2512_17073_b200/_lib
for v in ${@:-u2 u4 u1 u4 u2}; do
  cp $L/var_$v.so $L/liblrc.so
  for b in 1 8; do
    r=$(python bench.py --batch $b --no-sweep --no-prefill --no-offload --no-cpu-baseline --steps 2000 --warmup 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline'].get('phase_ms'))")
    echo "$v B=$b -> $r"
  done
done
