"""Full-opcode SASS histogram of one kernel (dev tool): python tools/sass_ops.py lib.so regex"""
import collections
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", out)[1:]:
    name = f.split("\n", 1)[0]
    if not re.search(sys.argv[2], name):
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9._]+)", f)
    c = collections.Counter(ins)
    print(name[:100], "total", len(ins))
    imad = sum(v for k, v in c.items() if k.startswith("IMAD"))
    wide = sum(v for k, v in c.items() if k.startswith("IMAD.WIDE"))
    print(f"   IMAD-class {imad} (WIDE {wide}); ", ", ".join(f"{k}:{v}" for k, v in c.most_common(24)))
