mkdir -p gpurun_out
for lv in 4 2 1 0; do
  echo "LO_LEVELS=$lv" >> gpurun_out/sw1.log
  LATSUM_LO_LEVELS=$lv SWEEP=0.10,0.11,0.12,0.13,0.14 timeout 600 python tools/profile_target.py atm_sweep >> gpurun_out/sw1.log 2>&1
done
