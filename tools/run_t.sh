mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t4_pytest.log 2>&1; echo rc=$? >> gpurun_out/t4_pytest.log
bash tools/ab_run.sh ab4.log base o1 head
