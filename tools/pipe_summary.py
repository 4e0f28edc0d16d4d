"""Per-kernel pipe utilisation and top warp-stall reasons from an ncu --page raw --csv export
(dev tool): python tools/pipe_summary.py raw.csv [title] > summary.txt"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[0], rows[2:]
title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
print(f"# source: {sys.argv[1]} ({title}); ncu --set full, one launch per row")
print("# pipe columns: % of peak sustained while the SM is active (sm__pipe_*_cycles_active / sm__inst_executed_pipe_lsu)")
cols = [("fp64", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("alu", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        ("fma", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("lsu", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        ("issue", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("us", "gpu__time_duration.sum")]
print(f"{'kernel':60s} " + " ".join(f"{c:>7s}" for c, _ in cols) + "  top stalls (cycles per issued instruction)")
for r in data:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "?")
    vals = []
    for c, k in cols:
        v = d.get(k, "")
        try:
            f = float(v.replace(",", ""))
            vals.append(f"{f / 1000 if c == 'us' and f > 1e4 else f:7.1f}")
        except ValueError:
            vals.append(f"{'-':>7s}")
    st = []
    for k, v in d.items():
        if "issue_stalled" in k and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v.replace(",", "")), k.split("issue_stalled_")[1].replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    print(f"{name[:60]:60s} " + " ".join(vals) + "  " + ", ".join(f"{n} {x:.2f}" for x, n in st[:4]))
