#!/usr/bin/env python
"""Summarise ptxas -v output of libgsde's kernels: one line per instantiation
(kernel, Cfg<STAR,SMEM,TAB,REFLECT,OCC,ZD,INJ> flags) with registers and spills.

    python tools/ptxas_summary.py [paper_2512_02175_b200/csrc/build/gsde_native.ptxas.txt] [filter]
"""
import re
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "paper_2512_02175_b200/csrc/build/gsde_native.ptxas.txt"
filt = sys.argv[2] if len(sys.argv) > 2 else ""
txt = open(path).read().splitlines()
name = None
for i, l in enumerate(txt):
    m = re.search(r"Function properties for (\S+)", l)
    if m:
        name = m.group(1)
        km = re.search(r"\d+((?:native|ref|fvm|histogram|step)\w*?_kernel)", name)
        flags = re.findall(r"Lb([01])E", name)
        ints = re.findall(r"Li(\d+)E", name)
        short = (km.group(1) if km else name[:40]) + "<" + "".join(flags) + ">" + (
            "[" + ",".join(ints) + "]" if ints else "")
        spill = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", txt[i + 1])
        regs = None
        for l2 in txt[i + 1:i + 4]:
            r = re.search(r"Used (\d+) registers", l2)
            if r:
                regs = r.group(1)
                break
        if filt in short:
            print(f"{short:60s} regs={regs} spill={spill.group(1)}/{spill.group(2)}")
