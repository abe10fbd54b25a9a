"""Opcode counts of the dispatched sm_100a kernels (cuobjdump -sass of the
built library): the evidence that the packed-FMA / MUFU paths are what runs.
    python tools/sass_summary.py [lib] > profiles/r02_sass_summary.txt"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

LIB = Path(sys.argv[1]) if len(sys.argv) > 1 else \
    Path(__file__).resolve().parent.parent / "paper_1812_07122_b200" / "_lib" / "libblfls.so"
KEYS = ["FFMA2", "FMUL2", "FADD2", "FFMA", "MUFU.EX2", "MUFU.RCP", "LDS", "STS", "LDG", "STG", "LDGSTS",
        "DFMA", "UBLKCP", "UTMALDG", "UTMASTG", "BAR", "SHFL", "ATOMS", "RED", "HMMA", "UTCHMMA"]
# kernels the c1-c5 workloads dispatch (launch list of the bench / smoke)
WANT = [r"k_blf_j3rILi7ELb0ELi12E", r"k_blf_p2rILi7ELb0ELi4ELb1E", r"k_blf_p2rILi15ELb0ELi4ELb1E", r"k_blf_p2rILi5ELb0ELi8ELb0E", r"k_col_triILi32ELi2ELi4ELi256E", r"k_blf_j3ILi7ELi32ELb0ELi2ELb1ELb1E", r"k_blf_p2ILi7ELi32ELi0ELi7ELb0ELi2ELb1ELb1E",
        r"k_blf_p2ILi15ELi16ELi0ELi5ELb0ELi4ELb1ELb1E", r"k_blf_p2ILi5ELi32ELi0ELi10ELb0ELi2ELb1ELb0E",
        r"k_row_r2cILb0ENS_5CtFftILi1024ELi2ELi128E", r"k2_colINS_4Fft2ILi2048ELi4ELi128ELi16E",
        r"k2_row_c2rINS_4Fft2ILi1024ELi4ELi64ELi16E", r"k2_row_c2r_tmaINS_4Fft2ILi1024ELi4ELi64ELi16E", r"k_grid_splat_tiled", r"k_dt_window"]

out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
print(f"# cuobjdump -sass {LIB.name} (sm_100a); opcode counts per kernel (static instructions)")
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not any(re.search(w, name) for w in WANT):
        continue
    ops = Counter()
    for line in f.splitlines():
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    ops[k if k != "MUFU.EX2" else k] += 1
                    break
    total = sum(1 for line in f.splitlines() if re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", line))
    print(f"\n{name}\n  instructions {total}: " + ", ".join(f"{k} {ops[k]}" for k in KEYS if ops[k]))
