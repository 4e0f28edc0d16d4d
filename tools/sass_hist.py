"""Per-function SASS instruction histogram of libckks.so (dev tool)."""
import collections
import re
import subprocess
import sys

so = sys.argv[1]
pat = sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if not re.search(pat, name):
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9._]+)", f)
    c = collections.Counter(i.split(".")[0] for i in ins)
    print(name[:110], "total", len(ins))
    print("   ", ", ".join(f"{k}:{v}" for k, v in c.most_common(18)))
