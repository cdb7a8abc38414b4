"""Summarise an ncu --metrics gpu__time_duration.sum launch list per kernel."""
import csv, sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    tot, cnt, mx = defaultdict(float), defaultdict(int), defaultdict(float)
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        us = float(d["Metric Value"].replace(",", "")) * scale
        tot[name] += us
        cnt[name] += 1
        mx[name] = max(mx[name], us)
    total = sum(tot.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s} {'max_us':>8s}")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k:40s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k]/total:6.1%} {tot[k]/cnt[k]:8.2f} {mx[k]:8.1f}")
    print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {total:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
