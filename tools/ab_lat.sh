#!/usr/bin/env bash
# A/B of library variants on several lattices: bash tools/ab_lat.sh LOG "fcc bcc" v1 v2 ...
LOG="gpurun_out/$1"; LATS="$2"; shift; shift
mkdir -p gpurun_out
for round in 1 2; do
  for lat in $LATS; do
    for v in "$@"; do
      if [ "$v" = "head" ]; then lib=""; else lib="paper_2504_11989_b200/_lib_ab/$v.so"; fi
      LATTICE=$lat AB_TAG="$lat $v" LATSUM_LIB="$lib" timeout 300 python tools/ab_time.py 20 >> "$LOG" 2>&1
    done
  done
done
