"""Key counters of one kernel from an ncu report: python tools/ncu_metrics.py rep.ncu-rep nodes out.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'sm__issue_active.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'smsp__inst_executed.sum',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio',
        'dram__bytes_read.sum', 'dram__bytes_write.sum']


def main(rep, units, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    res = {k: d.get(k) for k in KEYS}
    t = float(d['gpu__time_duration.sum']) * 1e-3 if d['gpu__time_duration.sum'] else None
    unit = rows[1][rows[0].index('gpu__time_duration.sum')]
    if unit in ('usecond', 'us'):
        t = float(d['gpu__time_duration.sum']) * 1e-6
    cyc = float(d['sm__cycles_elapsed.avg'])
    f = lambda k: float(d[k]) * cyc
    fl = 2 * f('smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed') + \
        f('smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed') + \
        f('smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed')
    res.update({'seconds': t, 'fp64_flops': fl, 'flops_per_unit': fl / float(units), 'tflops': fl / t / 1e12})
    for k, v in res.items():
        print(k, v)
    json.dump(res, open(out, 'w'), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:4])
