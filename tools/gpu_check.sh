#!/usr/bin/env bash
# One gpurun call: GPU tests + smoke, one ncu --set full capture of the ATM kernel (its counters
# become profiles/atm_kernel_current.json, which bench.py reads), the bench line (both arms) and
# the launch list of the bench command.  ncu reports are exported to CSV on the box.
# Usage (from the repo root, under gpurun):  bash tools/gpu_check.sh TAG [skip-tests] [skip-ncu] [c1]
TAG="${1:-run}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
  echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
fi
export_rep() {  # $1 = report path without .ncu-rep, $2 = output prefix
  ncu -i "$1.ncu-rep" --page raw --csv > "$2_raw.csv" 2>/dev/null
  ncu -i "$1.ncu-rep" --page source --csv --print-source sass > "$2_sass.csv" 2>/dev/null
  ncu -i "$1.ncu-rep" --page details --csv > "$2_details.csv" 2>/dev/null
}
if [ "$3" != "skip-ncu" ]; then
  timeout 300 python tools/profile_target.py atm > gpurun_out/${TAG}_atm_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_kernel -c 1 \
      -o /tmp/${TAG}_atm -f python tools/profile_target.py atm > gpurun_out/${TAG}_ncu_atm.log 2>&1
  export_rep /tmp/${TAG}_atm gpurun_out/${TAG}_atm
  python tools/ncu_metrics.py /tmp/${TAG}_atm.ncu-rep 25165824 gpurun_out/${TAG}_atm_metrics.json \
      > gpurun_out/${TAG}_atm_metrics.log 2>&1 && cp gpurun_out/${TAG}_atm_metrics.json profiles/atm_kernel_current.json
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
echo "ref rc=$?" >> gpurun_out/${TAG}_ref.err
if [ "$3" != "skip-ncu" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 1"
  timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
  if [ "$4" = "c1" ]; then
    timeout 300 python tools/profile_target.py c1 > gpurun_out/${TAG}_c1_plain.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -c 1 \
        -o /tmp/${TAG}_c1 -f python tools/profile_target.py c1 > gpurun_out/${TAG}_ncu_c1.log 2>&1
    export_rep /tmp/${TAG}_c1 gpurun_out/${TAG}_c1
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -s 2 -c 1 \
        -o /tmp/${TAG}_c1s -f python tools/profile_target.py c1_small > gpurun_out/${TAG}_ncu_c1s.log 2>&1
    export_rep /tmp/${TAG}_c1s gpurun_out/${TAG}_c1s
  fi
fi
du -sh gpurun_out/* | sort -h | tail -5 > gpurun_out/${TAG}_sizes.txt
echo done > gpurun_out/${TAG}_done
