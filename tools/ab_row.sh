#!/usr/bin/env bash
# A/B of the row-factorised ATM kernel across splits (one gpurun call): bash tools/ab_row.sh LOG
LOG="${1:-ab_row.log}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${LOG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${LOG}_pytest.log
bash tools/ab_env.sh $LOG "line1_0.13:LATSUM_LINE=1 LATSUM_ATM_SPLIT_SCALE=0.13" \
  "row_0.13:LATSUM_ATM_SPLIT_SCALE=0.13" "row_0.10:LATSUM_ATM_SPLIT_SCALE=0.10" \
  "row_0.08:LATSUM_ATM_SPLIT_SCALE=0.08" "row_0.06:LATSUM_ATM_SPLIT_SCALE=0.06" \
  "row_0.05:LATSUM_ATM_SPLIT_SCALE=0.05" "row_0.04:LATSUM_ATM_SPLIT_SCALE=0.04" \
  "row_0.03:LATSUM_ATM_SPLIT_SCALE=0.03"
