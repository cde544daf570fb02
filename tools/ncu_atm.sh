#!/usr/bin/env bash
# ncu --set full capture of one ATM kernel launch, exported to CSV (raw + SASS source page):
#   bash tools/ncu_atm.sh TAG
TAG="${1:-atm}"
mkdir -p gpurun_out
timeout 300 python tools/profile_target.py atm > gpurun_out/${TAG}_atm_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_kernel -c 1 \
    -o /tmp/${TAG}_atm -f python tools/profile_target.py atm > gpurun_out/${TAG}_ncu_atm.log 2>&1
ncu -i /tmp/${TAG}_atm.ncu-rep --page raw --csv > gpurun_out/${TAG}_atm_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_atm.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_atm_sass.csv 2>/dev/null
