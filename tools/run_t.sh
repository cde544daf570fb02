mkdir -p gpurun_out
LATSUM_LIB=paper_2504_11989_b200/_lib_ab/c1a.so timeout 900 python -m pytest tests/test_gpu_zeta.py tests/test_gpu_properties.py -q -m gpu -x > gpurun_out/c1a_pytest.log 2>&1; echo rc=$? >> gpurun_out/c1a_pytest.log
for r in 1 2; do for v in c1base c1a; do echo "== $v" >> gpurun_out/c1ab.log; LATSUM_LIB=paper_2504_11989_b200/_lib_ab/$v.so timeout 300 python tools/profile_target.py c1_time >> gpurun_out/c1ab.log 2>&1; done; done
