mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t17_pytest.log 2>&1; echo rc=$? >> gpurun_out/t17_pytest.log
for r in 1 2; do for v in c1prev head; do echo "== $v" >> gpurun_out/c1ab3.log; if [ $v = head ]; then lib=""; else lib=paper_2504_11989_b200/_lib_ab/$v.so; fi; LATSUM_LIB=$lib timeout 300 python tools/profile_target.py c1_time 2>&1 | grep -v lanes >> gpurun_out/c1ab3.log; done; done
