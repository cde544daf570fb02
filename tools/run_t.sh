mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_integrals.py -q -m gpu -x > gpurun_out/t7_pytest.log 2>&1; echo rc=$? >> gpurun_out/t7_pytest.log
bash tools/ab_env.sh ab7.log "head:X=1" "wpc24:LATSUM_LINE_WPC=24" "unr2:LATSUM_LINE_UNR=2" "w24u2:LATSUM_LINE_WPC=24 LATSUM_LINE_UNR=2"
