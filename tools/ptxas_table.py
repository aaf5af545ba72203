"""Per-kernel registers / stack / spills from `nvcc -Xptxas -v` (dev aid).
usage: python tools/ptxas_table.py csrc/sweep.cu"""
import re, subprocess, sys
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
                      "-Xcompiler", "-fPIC", "-c", sys.argv[1], "-o", "/tmp/_pt.o", "-Xptxas", "-v"],
                     capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        st = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur[:60]:60s} regs {m.group(1):>4s} stack {st[0]:>5s} spill st {st[1]:>5s} ld {st[2]:>5s}")
        cur = None
