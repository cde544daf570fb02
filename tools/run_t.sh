mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_integrals.py -q -m gpu -x > gpurun_out/t5_pytest.log 2>&1; echo rc=$? >> gpurun_out/t5_pytest.log
bash tools/ab_run.sh ab5.log base o1 head
