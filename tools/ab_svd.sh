#!/bin/bash
# A/B of svd_of_r (n = 128, 256; with and without V) and the C5 bench step across
# libraries / environment settings.
# usage: tools/ab_svd.sh "ENV=.. lib1.so" ["lib2.so" ...]
for spec in "$@"; do
  L=${spec##* }; E=""; [ "$L" != "$spec" ] && E=${spec% *}
  for n in 128 256; do for v in 1 0; do
    echo "$spec $(env $E JOINQR_LIB=$L timeout 120 python tools/svd_probe.py --n $n --vectors $v --reps 10 2>&1 | tail -1) vectors=$v"
  done; done
  env $E JOINQR_LIB=$L timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$spec C5 ms_per_step', d['ms_per_step'])"
done
