"""ptxas -v summary: one line per kernel (registers, spill bytes).
usage: python tools/ptxas_regs.py csrc/file.cu [name-filter]"""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cmd = ["nvcc", "-O3", "-std=c++17", "--expt-relaxed-constexpr", "-Iinclude", "-Ipaper_2010_15491_b200/csrc",
       "-gencode", "arch=compute_100a,code=sm_100a", "-Xptxas", "-v", "-c", src, "-o", "/tmp/_ptxas.o"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
res = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        res.setdefault(cur, {})["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        res.setdefault(cur, {})["regs"] = m.group(1)
for k, v in res.items():
    dm = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    if flt in dm:
        print(f"{v.get('regs','?'):>4} regs  spill {v.get('spill','?'):>10}  {dm[:150]}")
