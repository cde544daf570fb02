"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: time share per kernel."""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0][:70]
        v = float(r[idx["Metric Value"]].replace(",", "")) * SCALE.get(r[idx["Metric Unit"]], 1.0)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print("| kernel | launches | total ms | share | ms/launch |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / s:.2f}% | {v / cnt[k]:.4f} |")


if __name__ == "__main__":
    main(sys.argv[1])
