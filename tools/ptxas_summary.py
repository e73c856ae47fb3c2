"""ptxas_summary.py LOG [filter] -- registers / spills / smem per kernel from a -Xptxas -v log."""
import re
import subprocess
import sys

txt = open(sys.argv[1]).read()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
rows = {}
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = m.group(1)
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
for n, d in zip(names, dem):
    d = re.sub(r"\(.*", "", d.replace("(anonymous namespace)::", ""))
    if flt in d:
        print(f"{rows[n].get('regs', '?'):>4} regs  spill {rows[n].get('spill', '?'):>9}  {d}")
