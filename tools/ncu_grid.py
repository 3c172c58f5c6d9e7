"""Per-(kernel, grid) breakdown of an ncu --csv launch list with time + dram bytes."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if r and r[0] == "ID"][0]
per = collections.defaultdict(dict); info = {}
for r in rows:
    if r and r[0] != "ID" and len(r) == len(hdr):
        d = dict(zip(hdr, r)); i = d["ID"]; info[i] = (d["Kernel Name"][:34], d["Grid Size"])
        per[i][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for kname in sys.argv[2:]:
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        if kname in info[i][0]:
            a = agg[info[i][0][:28] + " " + info[i][1]]; a[0] += 1
            a[1] += m["gpu__time_duration.sum"] / 1e3
            a[2] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
    print(kname)
    for g, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"   {g:48s} n={n:3d} t={t:8.1f}us avg {t/n:6.1f}us {b/n:7.1f}MB {b/t*1e3 if t else 0:6.0f} GB/s")
