#!/usr/bin/env python
"""Dump SASS of the hot kernels of libucp_b200.so into profiles/ and print
the instruction mix that proves the vector path (LDG.E.NA.128 / STG.E.128,
no local-memory spills)."""
import re
import subprocess
import sys

LIB = "paper_2406_18820_b200/libucp_b200.so"
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", txt)
out = []
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    m = re.search(r"(convert_gather_\w+?|load_scatter_\w+?|reshard_fused_\w+?|adam_step_kernel|"
                  r"gen_state_kernel|compare_kernel)E", name)
    short = m.group(1) if m else name
    body = f
    mix = {k: len(re.findall(k, body)) for k in (r"LDG\.E\.NA\.128", r"LDG\.E\.128", r"STG\.E\.128",
                                                 r"STG\.E\.64", r"\bSTL\b", r"\bLDL\b", r"DADD", r"DMUL")}
    out.append((short, mix))
    if any(k in name for k in ("convert_gather_f32", "load_scatter_bf16", "reshard_fused_f32",
                               "reshard_fused_bf16")):
        with open(f"profiles/sass_{short}_{tag}.txt", "w") as fh:
            fh.write("Function : " + f)
for n, m in out:
    print(n[:60].ljust(60), m)
