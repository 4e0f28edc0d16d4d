"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into per-kernel shares."""
import collections
import csv
import re
import sys


def short(name: str) -> str:
    name = re.sub(r"^void\s+", "", name)
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", name)
    base = re.split(r"[<(]", name, 1)[0].split("::")[-1]
    m = re.search(r"k_elem<\s*(\w+)", name)
    if base == "k_elem" and m:
        base += ":" + m.group(1)
    m = re.search(r"k_fwd_cols(?:_f64)?<\s*\d+,\s*(?:\d+,\s*)?(\w+)", name)
    if base in ("k_fwd_cols", "k_fwd_cols_f64") and m:
        base += ":" + m.group(1)
    return base


def main(path, skip_torch=True):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        n = short(r[ki])
        if skip_torch and not n.startswith("k_"):
            continue
        tot[n] += float(r[vi].replace(",", ""))
        cnt[n] += 1
    s = sum(tot.values())
    print(f"libckks launches: {sum(cnt.values())}, summed device time {s / 1e6:.3f} ms (cold-cache, serialised)")
    print(f"{'kernel':34s} {'launches':>8s} {'share':>7s} {'avg us':>9s}")
    for k, v in tot.most_common():
        print(f"{k:34s} {cnt[k]:8d} {v / s * 100:6.2f}% {v / cnt[k] / 1e3:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
