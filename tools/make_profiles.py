"""Write text summaries of ncu reports / launch lists into profiles/ (tracked)."""
import io
import os
import subprocess
import sys
from contextlib import redirect_stdout

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import launch_shares  # noqa: E402
import ncu_summary  # noqa: E402

STALL_PREFIX = "smsp__average_warps_issue_stalled_"


def stalls(rep):
    import csv
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    out = []
    for i, m in enumerate(h):
        if m.startswith(STALL_PREFIX) and m.endswith("per_issue_active.ratio"):
            try:
                v = float(rows[2][i])
            except ValueError:
                continue
            if v > 0.05:
                out.append((v, m[len(STALL_PREFIX):]))
    return sorted(out, reverse=True)


def main(out_dir, items):
    os.makedirs(out_dir, exist_ok=True)
    for src, name in items:
        buf = io.StringIO()
        with redirect_stdout(buf):
            if src.endswith(".csv"):
                launch_shares.main(src)
            else:
                ncu_summary.run(src)
                print("\n   warp stall reasons (cycles per issued instruction):")
                for v, m in stalls(src):
                    print(f"   {m:70s} {v:.3f}")
        open(os.path.join(out_dir, name), "w").write(f"# source: {src}\n" + buf.getvalue())
        print("wrote", name)


if __name__ == "__main__":
    args = sys.argv[2:]
    main(sys.argv[1], list(zip(args[0::2], args[1::2])))
