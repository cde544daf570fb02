"""Static SASS loop report: every backward branch (loop) with its body size and opcode mix.

    cuobjdump -sass -fun <mangled> lib.o > k.sass; python tools/sass_loops.py k.sass
"""
import collections
import re
import sys

pat = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
ins = []
for line in open(sys.argv[1]):
    m = pat.search(line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
min_len = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA(?:\.\w+)*\s+(?:`\()?\.?L?_?x?_?(0x[0-9a-f]+|\w+)", txt)
    if "BRA" not in txt:
        continue
    tgt = re.findall(r"0x([0-9a-f]+)", txt)
    if not tgt:
        continue
    t = int(tgt[-1], 16)
    if t in addr and addr[t] < i and i - addr[t] >= min_len:
        body = ins[addr[t]:i + 1]
        mix = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0] for _, s in body)
        fp = sum(v for k, v in mix.items() if k in ("DFMA", "DADD", "DMUL"))
        print("loop %#06x..%#06x: %d instr, fp64 %d (%.0f%%): %s" % (
            t, a, len(body), fp, 100.0 * fp / len(body),
            ", ".join("%s %d" % kv for kv in mix.most_common(14))))
