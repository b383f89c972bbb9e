"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    out = []
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
              "s": 1e6}.get(u, 1.0)
        out.append((d["Kernel Name"], d["Grid Size"], d["Block Size"], v))
    return out


def short(name):
    name = re.sub(r"\(.*$", "", name.replace("void ", ""))
    return name[:100]


def main(path, skip_re=None):
    L = load(path)
    agg = collections.OrderedDict()
    for name, grid, block, us in L:
        if skip_re and re.search(skip_re, name):
            continue
        k = (short(name), grid)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"{len(L)} launches, {tot:.1f} us total (excluding {skip_re})")
    for (k, grid), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:5d} {t:10.1f} us {100 * t / tot:5.1f}%  avg {t / c:8.2f}  {grid:>14s}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
