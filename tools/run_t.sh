mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t9_pytest.log 2>&1; echo rc=$? >> gpurun_out/t9_pytest.log
timeout 900 python tools/profile_target.py adaptive_fcc > gpurun_out/t9_adaptive.log 2>&1
