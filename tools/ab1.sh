mkdir -p gpurun_out
for v in 20 24 16; do for u in 1 2; do
  AB_TAG="wpc$v unr$u" LATSUM_LINE_WPC=$v LATSUM_LINE_UNR=$u timeout 300 python tools/ab_time.py >> gpurun_out/ab1.log 2>&1
done; done
AB_TAG="wpc20 unr1 again" timeout 300 python tools/ab_time.py >> gpurun_out/ab1.log 2>&1
