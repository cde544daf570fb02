"""Key counters of one kernel launch from an ncu report (the roofline inputs of bench.py).

    python tools/ncu_metrics.py rep.ncu-rep UNITS out.json [KERNEL_NAME]

UNITS = algorithmic units (quadrature nodes) the captured launch processed.  FP64 FLOPs =
2 DFMA + DADD + DMUL thread instructions.  The output also records the sha1 of
csrc/kernels.cu at capture time so bench.py can tell a stale capture from the shipping build;
copy it to profiles/atm_kernel_current.json to make it the one bench.py reads.
"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ['gpu__time_duration.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'sm__issue_active.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'smsp__inst_executed.sum',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio',
        'dram__bytes_read.sum', 'dram__bytes_write.sum']
_SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
          "msecond": 1e-3, "second": 1.0}


def main(rep, units, out, kernel=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, unit_row = rows[0], rows[1]
    row = rows[2]
    if kernel:
        name_col = head.index("Kernel Name")
        row = next(r for r in rows[2:] if kernel in r[name_col])
    d = dict(zip(head, row))
    u = dict(zip(head, unit_row))

    def val(k):
        return float(d[k].replace(",", "")) * _SCALE.get(u.get(k, ""), 1.0)

    secs = val('gpu__time_duration.sum')
    cyc = float(d['sm__cycles_elapsed.avg'].replace(",", ""))
    f = lambda k: float(d[k].replace(",", "")) * cyc
    fl = 2 * f('smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed') + \
        f('smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed') + \
        f('smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed')
    sha = hashlib.sha1()
    for name in ("kernels.cu", "lz_internal.h", "special.cuh", "capi.cpp", "context.cpp"):
        sha.update(open(os.path.join(ROOT, "paper_2504_11989_b200", "csrc", name), "rb").read())
    res = {"kernel": d.get("Kernel Name"), "source": f"ncu --set full capture {os.path.basename(rep)}",
           "seconds": secs, "fp64_flops_per_launch": fl, "units_per_launch": float(units),
           "flops_per_unit": fl / float(units), "tflops": fl / secs / 1e12,
           "dram_bytes_per_launch": val('dram__bytes_read.sum') + val('dram__bytes_write.sum'),
           "fp64_pipe_active": val('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') / 100,
           "issue_active": val('sm__issue_active.avg.pct_of_peak_sustained_elapsed') / 100,
           "lsu_wavefronts": val('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed') / 100,
           "warps_active": val('sm__warps_active.avg.pct_of_peak_sustained_active') / 100,
           "registers": int(val('launch__registers_per_thread')),
           "csrc_sha1": sha.hexdigest(),
           "raw": {k: d.get(k) for k in KEYS}}
    for k, v in res.items():
        print(k, v)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:5])
