"""Instruction histogram of every loop body (backward branch) in one kernel's SASS."""
import collections
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", out)[1:]:
    name = f.split("\n", 1)[0]
    if not re.search(sys.argv[2], name):
        continue
    L = [l for l in f.splitlines() if re.search(r"/\*[0-9a-f]{4}\*/", l)]
    addr = lambda l: int(re.search(r"/\*([0-9a-f]{4})\*/", l).group(1), 16)
    for l in L:
        m = re.search(r"BRA.*?0x([0-9a-f]+)", l)
        if m and int(m.group(1), 16) < addr(l):
            lo, hi = int(m.group(1), 16), addr(l)
            body = [x for x in L if lo <= addr(x) <= hi]
            c = collections.Counter(re.search(r"\*/\s+(?:@!?U?P\w\s+)?([A-Z][A-Z0-9_.]*)", x).group(1) for x in body)
            heavy = sum(v * (2 if k.startswith("IMAD.WIDE") else 1) for k, v in c.items() if k.startswith("IMAD"))
            print(f"{name[:60]} loop {hex(lo)}-{hex(hi)}: {len(body)} instrs, heavy-pipe slots ~{heavy}")
            print("   ", ", ".join(f"{k}:{v}" for k, v in c.most_common(16)))
