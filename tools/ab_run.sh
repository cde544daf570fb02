#!/usr/bin/env bash
# A/B timing of library variants under one gpurun call: bash tools/ab_run.sh LOG v1 v2 ...
# (each variant paper_2504_11989_b200/_lib_ab/<v>.so; "head" = the in-tree library), two rounds
LOG="gpurun_out/$1"; shift
mkdir -p gpurun_out
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = "head" ]; then lib=""; else lib="paper_2504_11989_b200/_lib_ab/$v.so"; fi
    AB_TAG="$v" LATSUM_LIB="$lib" timeout 300 python tools/ab_time.py 20 >> "$LOG" 2>&1
  done
done
