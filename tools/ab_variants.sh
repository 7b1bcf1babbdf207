#!/bin/bash
# A/B timing of library variants (build/var/*.so) on the headline sweep:
# tools/ab_variants.sh base s1 k1 ...   ("base" = the in-tree library)
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=paper_1702_08880_b200/liblandau_b200.so; else lib=build/var/$v.so; fi
    t=$(LB_LIB=$lib python tools/prof_sweep.py 65536 6 | grep '^rep' | tail -4 | awk '{s+=$4} END {printf "%.3f", s/NR}')
    echo "round $round $v sweep_ms $t"
  done
done
