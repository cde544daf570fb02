mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t28_pytest.log 2>&1; echo rc=$? >> gpurun_out/t28_pytest.log
bash tools/ab_env.sh ab28.log "head:X=1" "c18:LATSUM_TABLE_CUTOFF=1e-18 LATSUM_DIRECT_CUTOFF=1e-18"
SWEEP=0.11,0.12,0.13,0.14,0.15 timeout 600 python tools/profile_target.py atm_sweep > gpurun_out/sw28.log 2>&1
