"""Build an A/B variant of the library with extra nvcc defines (tuning aid):

    python tools/build_variant.py NAME -DLZ_FOO=1 ...   -> paper_2504_11989_b200/_lib_ab/NAME.so

Run it with LATSUM_LIB=paper_2504_11989_b200/_lib_ab/NAME.so (tools/ab_time.py)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_11989_b200 import _native as N  # noqa: E402


def main(name, defines):
    out_dir = os.path.join(ROOT, "paper_2504_11989_b200", "_lib_ab")
    os.makedirs(out_dir, exist_ok=True)
    flags = [f for f in N.NVCC_FLAGS if f not in ("-shared", "-ldl")] + list(defines)
    srcs = [os.path.join(N.CSRC, s) for s in N.SOURCES]
    objs = [os.path.join(out_dir, f"{name}.{os.path.basename(s)}.o") for s in srcs]

    def one(pair):
        s, o = pair
        r = subprocess.run(["nvcc", *flags, "-c", s, "-o", o], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stdout + r.stderr)

    with ThreadPoolExecutor(len(srcs)) as pool:
        list(pool.map(one, zip(srcs, objs)))
    lib = os.path.join(out_dir, name + ".so")
    r = subprocess.run(["nvcc", *N.NVCC_FLAGS, *objs, "-o", lib], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stdout + r.stderr)
    for o in objs:
        os.remove(o)
    print(lib)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
