"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, mean / total device time and share (cold-cache, serialised
times: compare shares, not absolutes)."""
import collections
import csv
import sys


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    agg = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("unnamed>::", "")
        unit, val = r[13], float(r[14].replace(",", ""))
        us = val / 1e3 if unit in ("ns", "nsecond") else val * 1e3 if unit in ("ms", "msecond") else val
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':28s} {'launches':>8s} {'mean_us':>10s} {'total_us':>12s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:28s} {n:8d} {t / n:10.2f} {t:12.1f} {t / tot * 100:6.1f}%")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
