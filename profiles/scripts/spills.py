"""Registers / spills per kernel from /tmp/ptxas.log (dev helper): python spills.py REGEX"""
import re, subprocess, sys
pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
cur = None
regs = {}
for l in open("/tmp/ptxas.log"):
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip().split("(")[0]
    elif cur and pat.search(cur) and ("spill stores" in l or "Used" in l):
        regs.setdefault(cur, []).append(l.strip())
for k, v in regs.items():
    print(k[:80], " | ".join(x.replace("ptxas info    : ", "") for x in v)[:150])
