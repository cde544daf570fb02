mkdir -p gpurun_out
for i in 1 2 3 4; do timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rep$i.log 2>&1; echo "rc=$?" >> gpurun_out/rep$i.log; done
bash tools/gpu_check.sh r02h
