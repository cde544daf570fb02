"""Per-region instruction / stall / shared-wavefront shares of one kernel from an ncu SASS source
page: python tools/ncu_regions.py page.csv lo-hi:name [lo-hi:name ...]   (hex offsets)"""
import csv
import sys


def main(path, specs):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    col = {k: hdr.index(k) for k in ("Address", "Source", "Instructions Executed",
                                     "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared")}
    base = int(data[0][col["Address"]], 16)
    regions = []
    for sp in specs:
        rng, name = sp.split(":")
        lo, hi = (int(v, 16) for v in rng.split("-"))
        regions.append((lo, hi, name))
    keys = ("Instructions Executed", "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared")
    tot = {k: 0 for k in keys}
    acc = {r[2]: {k: 0 for k in keys} for r in regions}
    acc["other"] = {k: 0 for k in keys}
    for r in data:
        off = int(r[col["Address"]], 16) - base
        name = next((n for lo, hi, n in regions if lo <= off <= hi), "other")
        for k in keys:
            v = int(float(r[col[k]] or 0))
            tot[k] += v
            acc[name][k] += v
    print("%-16s %8s %8s %8s" % ("region", "inst", "stalls", "smem wf"))
    for name, a in acc.items():
        print("%-16s %7.1f%% %7.1f%% %7.1f%%" % (name, *(100.0 * a[k] / max(tot[k], 1) for k in keys)))
    print("totals", tot)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
