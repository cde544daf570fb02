#!/usr/bin/env bash
# A/B timing of env-var variants: bash tools/ab_env.sh LOG "TAG1:VAR=val VAR2=val" "TAG2:..." ...
LOG="gpurun_out/$1"; shift
mkdir -p gpurun_out
for round in 1 2; do
  for spec in "$@"; do
    tag="${spec%%:*}"; vars="${spec#*:}"
    env $vars AB_TAG="$tag" timeout 300 python tools/ab_time.py 20 >> "$LOG" 2>&1
  done
done
