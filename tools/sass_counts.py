"""SASS evidence for the psi pass: compiles psi.cu for sm_100a, finds the hot loop
of psi_kernel<8, r> (the 16 x unrolled 64-column chunk: the loop with the most MUFU.EX2), and
prints its opcode histogram and the instructions per pair (R = 8 rows x 64 columns = 512 pairs per
chunk per thread), plus an excerpt of the loop body.  No GPU needed.
usage: python tools/sass_counts.py > profiles/r02_sass_psi_kernel.txt"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1505_02100_b200", "csrc")


def sass_functions(cubin):
    txt = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True, check=True).stdout
    out = {}
    for f in re.split(r"\n\s+Function : ", txt)[1:]:
        name = f.split("\n")[0].strip()
        ops = []
        for line in f.split("\n"):
            m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", line)
            if m:
                ops.append((int(m.group(1), 16), m.group(3), line.strip()))
        out[name] = ops
    return out


def hot_loop(ops):
    best = None
    for i, (addr, op, _) in enumerate(ops):
        if op.startswith("BRA"):
            m = re.search(r"BRA\s+(?:`\()?0x([0-9a-f]+)", ops[i][2])
            if not m:
                continue
            tgt = int(m.group(1), 16)
            if tgt >= addr:
                continue
            j = next((k for k, o in enumerate(ops) if o[0] == tgt), None)
            if j is None:
                continue
            seg = ops[j:i + 1]
            mufu = sum(1 for o in seg if o[1].startswith("MUFU"))
            # the innermost loop that holds the chunk's 512 MUFU.EX2
            if mufu >= 512 and (best is None or len(seg) < len(best)):
                best = seg
    return best


def main():
    with tempfile.TemporaryDirectory() as td:
        cubin = os.path.join(td, "psi.cubin")
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-cubin",
                        "-I", os.path.join(ROOT, "include"), "-o", cubin, os.path.join(CSRC, "psi.cu")], check=True)
        funcs = sass_functions(cubin)
    for r in (6, 4):
        name = next(k for k in funcs if k.startswith(f"_ZN3plg10psi_kernelILi8ELi{r}E"))
        loop = hot_loop(funcs[name])
        c = Counter(o[1].split(".")[0] for o in loop)
        pairs = 8 * 64  # rows x columns per chunk per thread
        lane_ops = 2 * (c["FFMA2"] + c["FMUL2"] + c["FADD2"])  # packed: 2 lane-ops each
        print(f"== psi_kernel<8, {r}> hot loop (one 64-column chunk, 8 rows per thread = {pairs} pairs)")
        print(f"   instructions {len(loop)}; per pair: {len(loop) / pairs:.3f} issued, "
              f"MUFU.EX2 {c['MUFU'] / pairs:.3f}, FP32 lane-ops {lane_ops / pairs:.3f} "
              f"(FFMA2 {c['FFMA2']}, FMUL2 {c['FMUL2']}, FADD2 {c['FADD2']}), LDS {c['LDS']}")
        print("   histogram:", ", ".join(f"{k} {v}" for k, v in c.most_common()))
        print("   excerpt (first 40 instructions of the loop body):")
        for o in loop[:40]:
            print("     ", o[2])
        print()


if __name__ == "__main__":
    sys.exit(main())
