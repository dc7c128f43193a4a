"""Per-launch table (+ per-family summary, + mean GEMM DRAM bytes/launch) of the last step of an ncu
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv` launch list.
  python tools/launch_step_csv.py <ncu.csv> <launches_per_step> <out_prefix>"""
import collections, csv, json, re, sys

src, per, pre = sys.argv[1], int(sys.argv[2]), sys.argv[3]
lines = [l for l in open(src) if l.startswith('"')]
by = collections.OrderedDict()
for r in csv.DictReader(lines):
    d = by.setdefault(r["ID"], {"kernel": r["Kernel Name"], "grid": r.get("Grid Size", ""), "block": r.get("Block Size", "")})
    v = float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        d["time_us"] = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(r["Metric Unit"], 1.0)
    elif r["Metric Name"].startswith("dram__bytes"):
        d[r["Metric Name"].split(".")[0].replace("dram__bytes_", "dram_") + "_B"] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
rows = list(by.values())[-per:]
with open(pre + "_step.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["idx", "kernel", "grid", "block", "time_us", "dram_read_B", "dram_write_B"])
    for i, r in enumerate(rows):
        w.writerow([i, r["kernel"][:80], r["grid"], r["block"], round(r["time_us"], 3), int(r.get("dram_read_B", 0)), int(r.get("dram_write_B", 0))])
fam = collections.OrderedDict()
for r in rows:
    k = re.sub(r"\(.*", "", r["kernel"]).replace("void ", "").replace("pcpp::", "")[:44]
    a = fam.setdefault(k, [0, 0.0, 0.0]); a[0] += 1; a[1] += r["time_us"]; a[2] += r.get("dram_read_B", 0) + r.get("dram_write_B", 0)
tot = sum(a[1] for a in fam.values())
with open(pre + "_summary.txt", "w") as f:
    f.write(f"# {src}: last {per} launches (one step); cold-cache, serialised launches: compare shares, not absolutes\n")
    f.write(f"{'kernel':44s} {'launches':>8s} {'total us':>10s} {'mean us':>8s} {'share':>7s} DRAM MB/launch\n")
    for k, a in sorted(fam.items(), key=lambda x: -x[1][1]):
        f.write(f"{k:44s} {a[0]:8d} {a[1]:10.1f} {a[1] / a[0]:8.2f} {100 * a[1] / tot:6.1f}% {a[2] / a[0] / 1e6:10.2f}\n")
    f.write(f"{'TOTAL':44s} {len(rows):8d} {tot:10.1f}\n")
    g = [r for r in rows if "gemm_tc" in r["kernel"]]
    gb = sum(r.get("dram_read_B", 0) + r.get("dram_write_B", 0) for r in g) / max(len(g), 1)
    f.write(f"gemm_tc (all variants): {len(g)} launches, {sum(r['time_us'] for r in g):.1f} us, mean DRAM traffic {gb / 1e6:.2f} MB/launch\n")
json.dump({"source": f"{pre}_step.csv: ncu dram__bytes_read.sum + dram__bytes_write.sum per gemm_tc* launch of one 1024^2 step",
           "gemm_launches": len(g), "gemm_dram_bytes_per_launch": gb}, open(pre + "_gemm_traffic.json", "w"), indent=1)
