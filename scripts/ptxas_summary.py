#!/usr/bin/env python
"""Per-function ptxas summary (registers, stack, spills) of one .cu file.
Usage: scripts/ptxas_summary.py <file.cu> [-DX=..] [--filter substr]"""
import re, subprocess, sys
args = sys.argv[1:]
flt = None
if "--filter" in args:
    i = args.index("--filter"); flt = args[i + 1]; del args[i:i + 2]
src, extra = args[0], args[1:]
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
       "-std=c++17", "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", "include", "-c", src,
       "-o", "/tmp/ptxas_summary.o"] + extra
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    print(r.stderr[-4000:]); sys.exit(1)
names = set(re.findall(r"(?:for|function) '?(_Z\w+)", r.stderr))
dem = {}
if names:
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    dem = dict(zip(names, out))
def short(m):
    d = dem.get(m, m)
    d = re.sub(r"kcb::\(anonymous namespace\)::", "", d)
    d = re.sub(r"\(.*", "", d)
    return d.replace("void ", "")
cur = None; entry = None
for line in r.stderr.split("\n"):
    m = re.search(r"Compiling entry function '(_Z\w+)'", line)
    if m: entry = short(m.group(1)); continue
    m = re.search(r"Function properties for (_Z\w+)", line)
    if m: cur = short(m.group(1)); continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        st = (cur, m.groups()); 
        if flt is None or flt in (entry or ""):
            if int(m.group(1)) or int(m.group(2)) or int(m.group(3)) or cur == entry:
                print(f"  [{entry}] {cur}: stack {m.group(1)} spill st {m.group(2)} ld {m.group(3)}")
        continue
    m = re.search(r"Used (\d+) registers.*?(\d+ bytes smem)?", line)
    if m and (flt is None or flt in (entry or "")):
        print(f"[{entry}] regs {m.group(1)} {line.split('barriers')[-1].strip(', ')}")
