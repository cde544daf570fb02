#!/usr/bin/env bash
# A/B of library variants on the C1 zeta batches: bash tools/ab_c1.sh LOG v1 v2 ...
LOG="gpurun_out/$1"; shift
mkdir -p gpurun_out
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = "head" ]; then lib=""; else lib="paper_2504_11989_b200/_lib_ab/$v.so"; fi
    echo "== $v" >> "$LOG"
    LATSUM_LIB="$lib" timeout 300 python tools/profile_target.py c1_time >> "$LOG" 2>&1
  done
done
