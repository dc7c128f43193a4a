"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per kernel family,
launches and total/mean device time for the launches of ONE step (the last `per_step` rows)."""
import csv
import collections
import re
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    return [r for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]


def family(name):
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"<.*>", lambda m: m.group(0), n)
    return n.replace("pcpp::", "").strip()


def main(path, per_step=None):
    rows = load(path)
    if per_step:
        rows = rows[-per_step:]
    agg = collections.OrderedDict()
    for r in rows:
        f = family(r["Kernel Name"])
        t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)   # -> us
        a = agg.setdefault(f, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
    for f, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{f[:60]:60s} {n:8d} {t:10.1f} {t / n:9.2f} {100 * t / tot:5.1f}%")
    print(f"{'TOTAL':60s} {sum(v[0] for v in agg.values()):8d} {tot:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
