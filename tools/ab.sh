#!/bin/bash
# A/B timing helper (GPU box): tsqr_ms at m=2e6 for dense/footnote x n=32/64 (min of 5 reps)
# usage: tools/ab.sh [lib.so ...]
libs=("$@"); [ ${#libs[@]} -eq 0 ] && libs=(paper_2503_23385_b200/lib/libjoinqr.so)
for L in "${libs[@]}"; do
  for v in dense footnote; do for n in 32 64; do
    r=$(JOINQR_LIB=$L JOINQR_VARIANT=$v timeout 120 python tools/run_figaro.py --m 2000000 --n $n --reps 6 --all 2>&1 | tail -1)
    echo "$(basename $L) $v n=$n $r"
  done; done
done
