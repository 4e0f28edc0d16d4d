"""Summarise an ncu --page source --csv --print-source sass export: per kernel, executed
warp-instructions by opcode and warp-stall samples by reason (dev tool)."""
import collections
import csv
import gzip
import sys


def main(path, top=22):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    i = 0
    while i < len(rows):
        if rows[i] and rows[i][0] == "Kernel Name":
            name = rows[i][1]
            hdr = rows[i + 1]
            j = i + 2
            ins, samp, stall = collections.Counter(), collections.Counter(), collections.Counter()
            si = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
            while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
                r = dict(zip(hdr, rows[j]))
                opc = r["Source"].strip().split()
                if opc and opc[0].startswith("@"):
                    opc = opc[1:]
                o = opc[0].split(".")[0] if opc else "?"
                try:
                    ins[o] += int(r["Instructions Executed"] or 0)
                    samp[o] += int(r["# Samples"] or 0)
                except ValueError:
                    pass
                for k in si:
                    try:
                        stall[hdr[k]] += int(rows[j][k] or 0)
                    except ValueError:
                        pass
                j += 1
            tot = sum(ins.values())
            print(f"== {name[:100]}\n   warp-instructions executed: {tot}")
            print("   by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in ins.most_common(top)))
            ts = sum(stall.values())
            print("   stall samples:", ", ".join(f"{k[6:]} {v / ts:.1%}" for k, v in stall.most_common(10)))
            i = j
        else:
            i += 1


if __name__ == "__main__":
    main(sys.argv[1])
