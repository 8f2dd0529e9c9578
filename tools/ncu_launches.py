"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
total and mean device time, share of the total (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name)                 # drop parameter list
    name = name.replace("void ", "").replace("fgs::<unnamed>::", "").replace("fgs::", "")
    return name.strip()


def main(path, only_fgs=True):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        nm = short(r[iN])
        if only_fgs and ("at::" in nm or "elementwise" in nm or "reduce_kernel" in nm):
            continue
        v = float(r[iV].replace(",", ""))
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total us | mean us | share |")
    print(f"|---|---|---|---|---|")
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {c} | {v / 1e3:.1f} | {v / c / 1e3:.1f} | {100 * v / tot:.1f}% |")
    print(f"| **total** | {sum(c for c, _ in agg.values())} | {tot / 1e3:.1f} | | 100% |")


if __name__ == "__main__":
    main(sys.argv[1])
