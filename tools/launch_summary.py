"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import re
import sys


def summary(path, top=14):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    n = 0
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        try:
            v = float(r[idx["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        key = re.sub(r"\(.*", "", r[idx["Kernel Name"]])[:60]
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += v
        n += 1
    tot = sum(v[1] for v in agg.values())
    out = [f"{path}: {n} launches, {tot / 1e3:.1f} us total (ncu-serialised, cold caches)"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"  {k:60s} n={c:5d} {v / 1e3:10.1f} us  {100 * v / tot:5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summary(p))
