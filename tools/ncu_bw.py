"""Aggregate an ncu --csv launch list with time + dram bytes into per-kernel GB/s (markdown)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
SCALE = {"ns": 1e-3, "us": 1.0, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = collections.defaultdict(dict)
names = {}
for d in data:
    i = d["ID"]; names[i] = d["Kernel Name"]
    per[i][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i][:70]]
    a[0] += 1; a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"total {tot/1e3:.2f} ms over {len(per)} launches\n")
print("| kernel | launches | total (us) | share | DRAM MB | GB/s |\n|---|---|---|---|---|---|")
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"| {k} | {n} | {t:.1f} | {t/tot:.3f} | {b/1e6:.1f} | {b/1e3/t if t else 0:.0f} |")
