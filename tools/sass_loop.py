#!/usr/bin/env python3
"""Static SASS census of one kernel in libsphb200.so: instruction count, spills, and the
instruction mix of its innermost loops (backward branches), to check code quality on CPU
before spending GPU time.  usage: sass_loop.py <kernel-substring> [lib]"""
import re
import subprocess
import sys

name = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2604_12505_b200/libsphb200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    fname = f.split("\n", 1)[0].strip()
    if name not in fname:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print(f"== {fname}: {len(ins)} instructions, spills: "
          f"{sum('STL' in s for _, s in ins)} STL / {sum('LDL' in s for _, s in ins)} LDL")
    # loops: backward branches
    for addr, s in ins:
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", s)
        if m and m.group(1):
            tgt = int(m.group(1), 16)
            if tgt < addr:
                body = [x for a, x in ins if tgt <= a <= addr]
                mix = {}
                for x in body:
                    op = x.split()[0] if not x.startswith("@") else x.split()[1]
                    op = op.split(".")[0]
                    mix[op] = mix.get(op, 0) + 1
                top = sorted(mix.items(), key=lambda kv: -kv[1])[:12]
                print(f"  loop {tgt:#x}-{addr:#x}: {len(body)} instr, MUFU {mix.get('MUFU', 0)}, "
                      f"LDG {mix.get('LDG', 0)}, LDL {mix.get('LDL', 0)} | {top}")
