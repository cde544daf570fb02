mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t14_pytest.log 2>&1; echo rc=$? >> gpurun_out/t14_pytest.log
LATSUM_TIMING=1 timeout 300 python tools/profile_target.py e2e_breakdown > gpurun_out/e2e6.log 2>&1
