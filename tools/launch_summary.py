"""Aggregate an ncu launch-list CSV (gpu__time_duration.sum, dram bytes) by
kernel name: launches, total time, share, DRAM MB, achieved GB/s.

    python tools/launch_summary.py gpurun_out/resnet_launches.csv [top]
"""
import collections
import csv
import sys


def summarize(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = collections.defaultdict(lambda: [0, 0.0, 0.0])
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tmult = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name, m = d["Kernel Name"][:70], d["Metric Name"]
        v = float(d["Metric Value"].replace(",", ""))
        if m == "gpu__time_duration.sum":
            data[name][0] += 1
            data[name][1] += v * tmult.get(d["Metric Unit"], 1.0)
        elif m.startswith("dram__bytes"):
            data[name][2] += v * mult[d["Metric Unit"]]
    tot = sum(v[1] for v in data.values())
    out = [f"total {tot:.1f} us over {sum(v[0] for v in data.values())} launches", "",
           "| kernel | launches | total (us) | share | DRAM MB | GB/s |", "|---|---|---|---|---|---|"]
    for name, (n, t, b) in sorted(data.items(), key=lambda kv: -kv[1][1])[:top]:
        gbs = b / (t * 1e-6) / 1e9 if t else 0
        out.append(f"| {name} | {n} | {t:.1f} | {t / tot:.3f} | {b / 1e6:.1f} | {gbs:.0f} |")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30))
