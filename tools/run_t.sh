mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t8_pytest.log 2>&1; echo rc=$? >> gpurun_out/t8_pytest.log
bash tools/ab_run.sh ab8.log v4base horner rsq head p1u2
