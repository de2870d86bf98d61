#!/bin/bash
# usage: tools_ptxas_report.sh file.cu  -> kernel, regs, spills (demangled)
nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC -Xptxas -v -c "$1" -o /tmp/ptxas_report.o 2>&1 | python3 -c '
import sys, re, subprocess
lines = sys.stdin.read().splitlines()
cur = None
for i, l in enumerate(lines):
    m = re.search(r"Compiling entry function .(_Z\w+).", l) or re.search(r"Function properties for (_Z\w+)", l)
    if m: cur = m.group(1)
    m2 = re.search(r"(\d+) bytes spill stores", l)
    if m2: spill = m2.group(1)
    m3 = re.search(r"Used (\d+) registers", l)
    if m3 and cur:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"pftg::", "", name)
        name = re.sub(r"\(.*", "", name)
        print(f"{m3.group(1):>4} regs spill={spill:>5}  {name}")
'
