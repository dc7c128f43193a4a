"""Per (kernel, grid) breakdown of the last `per_step` launches of an ncu launch-list CSV."""
import csv, collections, sys
path = sys.argv[1]; per = int(sys.argv[2]) if len(sys.argv) > 2 else None
lines = [l for l in open(path) if l.startswith('"')]
rows = [r for r in csv.DictReader(lines) if r["Metric Name"] == "gpu__time_duration.sum"]
if per: rows = rows[-per:]
d = collections.defaultdict(list)
for r in rows:
    d[(r["Kernel Name"][:44], r.get("Grid Size", ""))].append(float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1))
for (k, g), v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:44s} {g:15s} n={len(v):3d} tot={sum(v):8.1f}us mean={sum(v)/len(v):7.2f} min={min(v):7.2f} max={max(v):7.2f}")
