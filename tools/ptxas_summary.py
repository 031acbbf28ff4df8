"""Summarise build/ptxas.log: registers / spills / smem per kernel."""
import re, subprocess, sys
log = open(sys.argv[1] if len(sys.argv) > 1 else "build/ptxas.log").read().splitlines()
cur = None
for i, line in enumerate(log):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(anonymous namespace\)::", "", cur)
        cur = cur.split("(")[0]
        continue
    m = re.search(r"Used (\d+) registers.*?(\d+) bytes smem", line)
    if m and cur:
        sp = re.search(r"(\d+) bytes spill stores", log[i - 1])
        print(f"{cur:45s} regs={m.group(1):>4} smem={m.group(2):>6} spill={sp.group(1) if sp else '?'}")
        cur = None
