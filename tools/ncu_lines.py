"""Per-source-line shares (instructions, stall samples, shared-memory wavefronts) of one kernel:
python tools/ncu_lines.py sass_page.csv nvdisasm_gi.sass kernel_substring source.cu [N [sortcol]]
(sass_page: ncu -i rep --page source --csv --print-source sass; nvdisasm_gi: nvdisasm -gi -c cubin).
Inlined one-line helpers (inline asm loads/stores) are charged to their call site."""
import collections
import csv
import re
import sys


def main(page, dis, kname, src, top=40):
    lines = open(dis).read().split("\n")
    start = [i for i, l in enumerate(lines) if l.startswith("//---") and kname in l][0]
    text = open(src).read().split("\n")
    helper = lambda ln: 0 < ln <= len(text) and "asm volatile" in text[ln - 1]
    cur, chain, off2line = None, [], {}
    for l in lines[start + 1:]:
        if l.startswith("//---"):
            break
        m = re.search(r'//## File ".*?", line (\d+)(?: inlined at ".*?", line (\d+))?', l)
        if m:
            chain.append(int(m.group(1)))
            if m.group(2):
                chain.append(int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            if chain:
                cur = next((ln for ln in chain if not helper(ln)), chain[0])
                chain = []
            if cur is not None:
                off2line[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(page)))
    hdr, data = rows[1], rows[2:]
    col = {k: hdr.index(k) for k in ("Address", "Instructions Executed", "Warp Stall Sampling (All Samples)",
                                     "L1 Wavefronts Shared")}
    base = int(data[0][col["Address"]], 16)
    acc = collections.defaultdict(lambda: [0, 0, 0])
    tot = [0, 0, 0]
    for r in data:
        ln = off2line.get(int(r[col["Address"]], 16) - base, -1)
        for j, k in enumerate(("Instructions Executed", "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared")):
            v = int(float(r[col[k]] or 0))
            acc[ln][j] += v
            tot[j] += v
    print("line   inst%  stall%  smemwf%  source")
    for ln, v in sorted(acc.items(), key=lambda kv: -kv[1][int(sys.argv[6]) if len(sys.argv) > 6 else 0])[:int(top)]:
        print("%5d %6.1f %7.1f %8.1f  %s" % (ln, *(100.0 * v[j] / max(tot[j], 1) for j in range(3)),
                                             text[ln - 1].strip()[:80] if ln > 0 else "?"))


if __name__ == "__main__":
    main(*sys.argv[1:6])
