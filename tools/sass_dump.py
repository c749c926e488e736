#!/usr/bin/env python
"""Dump SASS of every shipped kernel of libucp_b200.so into profiles/ and
print the instruction mix that proves the vector path (LDG.E.NA.128 /
STG.E.128, funnel shuffles for the realigning kernels, no local-memory
spills).

    python tools/sass_dump.py TAG        # writes profiles/sass_<kernel>_<TAG>.txt
"""
import re
import subprocess
import sys

LIB = "paper_2406_18820_b200/libucp_b200.so"
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", txt)
MIX = {"LDG.NA.128": r"LDG\.E\.NA\.128", "LDG.128": r"LDG\.E\.128", "LDG.NA.32": r"LDG\.E\.NA ",
       "STG.128": r"STG\.E\.128", "STG.64": r"STG\.E\.64", "STG.32": r"STG\.E(\.U16)? ",
       "SHFL.IDX": r"SHFL\.IDX", "STS.128": r"STS\.128", "LDS": r"LDS[ .]", "F2FP": r"F2FP",
       "STL": r"\bSTL\b", "LDL": r"\bLDL\b", "DADD": r"DADD", "DMUL": r"DMUL"}
rows = []
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    m = re.search(r"(convert_gather_\w+?|load_scatter_\w+?|reshard_fused_\w+?|adam_step_kernel|"
                  r"gen_state_kernel|compare_kernel|runtile_scan_kernel)E", name)
    if not m:
        continue
    short = m.group(1)
    mix = {k: len(re.findall(v, f)) for k, v in MIX.items()}
    n_instr = len(re.findall(r"/\*[0-9a-f]{4,}\*/", f))
    rows.append((short, n_instr, mix))
    with open(f"profiles/sass_{short}_{tag}.txt", "w") as fh:
        fh.write("Function : " + f)
for n, ni, m in sorted(rows):
    print(n.ljust(26), str(ni).rjust(6), {k: v for k, v in m.items() if v})
