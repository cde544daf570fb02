"""Instruction / stall / shared-wavefront shares of a kernel by straight-line SASS segment (runs of
instructions with the same execution count) from an ncu source page exported as CSV, plus a few
raw-page counters:  python tools/sass_segments.py page_sass.csv [page_raw.csv] [min_share_pct]"""
import csv
import sys


def main(sass, raw=None, min_share=0.4):
    rows = list(csv.reader(open(sass)))
    hdr, data = rows[1], rows[2:]
    ci = {k: hdr.index(k) for k in ["Address", "Source", "Instructions Executed",
                                    "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared", "stall_long_sb"]}
    base = int(data[0][0], 16)
    tot_i = sum(int(r[ci["Instructions Executed"]] or 0) for r in data)
    tot_s = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    tot_w = sum(int(float(r[ci["L1 Wavefronts Shared"]] or 0)) for r in data)
    segs = []
    for r in data:
        off = int(r[0], 16) - base
        n = int(r[ci["Instructions Executed"]] or 0)
        s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        w = int(float(r[ci["L1 Wavefronts Shared"]] or 0))
        lsb = int(r[ci["stall_long_sb"]] or 0)
        src = r[ci["Source"]]
        fp = any(t in src for t in ("DFMA", "DADD", "DMUL"))
        loc = any(t in src for t in ("LDL", "STL"))
        if segs and segs[-1][2] == n:
            g = segs[-1]
            g[1] = off; g[3] += 1; g[4] += s; g[5] += w; g[6] += fp; g[7] += lsb; g[8] += loc
        else:
            segs.append([off, off, n, 1, s, w, int(fp), lsb, int(loc)])
    print(f"instructions {tot_i}  stall samples {tot_s}  fp64 instr {sum(g[2]*g[6] for g in segs)}")
    for a, b, n, c, s, w, fp, lsb, loc in segs:
        share = n * c / tot_i * 100
        if share > float(min_share) or s / tot_s > 0.01:
            print(f"{a:#8x}-{b:#8x} exec {n:>9} x{c:>4}  inst {share:5.1f}%  stalls {s/tot_s*100:5.1f}% (long_sb {lsb/tot_s*100:4.1f}%)"
                  f"  smem wf {w/max(tot_w,1)*100:5.1f}%  fp64 {fp:>3} local {loc}")
    if raw:
        rr = list(csv.reader(open(raw)))
        d = dict(zip(rr[0], rr[2] if len(rr) > 2 else rr[1]))
        for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                  "launch__registers_per_thread", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                  "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                  "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                  "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
                  "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
                  "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
                  "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
                  "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
                  "sm__icc_request_hit_rate.pct", "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
                  "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
                  "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"):
            if k in d:
                print(f"  {k} = {d[k]}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
