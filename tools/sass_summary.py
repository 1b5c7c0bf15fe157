"""Per-kernel SASS instruction counts of the built library (cuobjdump -sass): the evidence that
the hot kernels are hand-written sm_100a code on the intended pipes — DMMA.8x8x4 fed by
UTMALDG (TMA) with SYNCS (mbarrier) for the tiled DGEMM, DMUL/DADD (no DFMA) for the bit-exact
modes, FMUL/FADD (no FFMA) with 128-bit LDG/STG for AXPY. Usage: python tools/sass_summary.py [so]"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OPS = ["DMMA", "UTMALDG", "UTMAPF", "SYNCS", "DFMA", "DMUL", "DADD", "FFMA", "FMUL", "FADD", "LDS", "LDG", "STG",
       "LDGSTS", "USETMAXREG", "BAR"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_1602_08477_b200" / "libkw_b200.so")
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)((?:\.[A-Za-z0-9_]+)*)", line)
        if m:
            op, mods = m.group(1), m.group(2)
            kernels[cur][op] += 1
            kernels[cur][op + mods] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.split("\n")
    print(f"# SASS instruction counts per kernel (static, cuobjdump -sass {Path(so).name}); opcode families:")
    print("# " + " ".join(OPS) + "  (+ the full opcode.modifier forms of DMMA / LDG / STG / UTMALDG)")
    for (name, cnt), dn in zip(kernels.items(), demangled):
        fam = {o: cnt.get(o, 0) for o in OPS if cnt.get(o, 0)}
        detail = {k: v for k, v in cnt.items() if "." in k and k.split(".")[0] in ("DMMA", "LDG", "STG", "UTMALDG")}
        short = re.sub(r"\(.*", "", dn.replace("(anonymous namespace)::", ""))
        print(f"{short[:150]}\n    {fam}\n    {detail}")


if __name__ == "__main__":
    main()
