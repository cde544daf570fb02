mkdir -p gpurun_out
for v in prev head; do
  if [ $v = head ]; then lib=""; else lib=paper_2504_11989_b200/_lib_ab/$v.so; fi
  LATSUM_LIB=$lib timeout 300 python tools/profile_target.py atm > /dev/null 2>&1
  LATSUM_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_kernel -c 1 -o /tmp/seg_$v -f python tools/profile_target.py atm > gpurun_out/seg_$v.log 2>&1
  ncu -i /tmp/seg_$v.ncu-rep --page raw --csv > gpurun_out/seg_${v}_raw.csv 2>/dev/null
  ncu -i /tmp/seg_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/seg_${v}_sass.csv 2>/dev/null
done
