"""SASS instruction census of libsemimat_b200.so (development aid; writes profiles/sass_census.txt).

Counts, per kernel, the opcodes that show which hardware path each kernel takes:
packed-integer lane updates (VIMNMX.U16x2 / VIADDMNMX.U16x2 and the 32-bit
forms), tcgen05 (UTCIMMA for kind::i8, UTCOMMA for the block-scaled kind::mxf4, LDTM, UTCBAR), TMA tensor loads (UTMALDG), 1-D bulk
async copies (UBLKCP), mbarrier ops (SYNCS.*), shared/global vector loads.
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
LIB = REPO / "paper_1705_08743_b200" / "libsemimat_b200.so"
OPS = ["VIMNMX.U16x2", "VIADDMNMX.U16x2", "VIMNMX", "VIADDMNMX", "IMNMX", "UTCIMMA", "UTCOMMA", "UTMALDG", "UBLKCP", "LDTM",
       "UTCBAR", "SYNCS.ARRIVE.TRANS64", "SYNCS.PHASECHK.TRANS64.TRYWAIT", "LDS.128", "LDG.E.128", "LOP3.LUT",
       "SHFL.IDX", "BAR.SYNC"]


def census(lib: Path):
    out = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs.setdefault(cur, Counter())
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)", line)
        if m and cur:
            op = m.group(1)
            for want in OPS:
                if op == want or op.startswith(want + "."):
                    funcs[cur][want] += 1
                    break
    return funcs


def main():
    funcs = census(LIB)
    lines = ["# SASS instruction census of libsemimat_b200.so (cuobjdump -sass, sm_100a; tools/sass_census.py)",
             "# opcodes: " + " ".join(OPS)]
    for name in sorted(funcs):
        c = funcs[name]
        if not c:
            continue
        lines.append(name)
        lines.append("    " + " ".join(f"{op}={c[op]}" for op in OPS if c[op]))
    text = "\n".join(lines) + "\n"
    dest = REPO / "profiles" / "sass_census.txt"
    dest.write_text(text)
    sys.stdout.write(text)


if __name__ == "__main__":
    main()
