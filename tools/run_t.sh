mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t12_pytest.log 2>&1; echo rc=$? >> gpurun_out/t12_pytest.log
LATSUM_TIMING=1 timeout 300 python tools/profile_target.py e2e_breakdown > gpurun_out/e2e5.log 2>&1
timeout 900 python bench.py --no-secondary > gpurun_out/b12.json 2> gpurun_out/b12.err
