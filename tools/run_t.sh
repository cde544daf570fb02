mkdir -p gpurun_out
for i in 1 2 3 4 5; do
  timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t26_$i.log 2>&1; echo rc=$? >> gpurun_out/t26_$i.log
done
