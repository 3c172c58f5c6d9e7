"""Summarise gpurun_out ncu artefacts into profiles/ (tracked)."""
import collections, csv, json, subprocess, sys

def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"]) * (1e3 if d.get("Metric Unit") == "usecond" else 1)
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = ["| kernel | launches | total (us) | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        out.append(f"| {k[:60]} | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / tot:.3f} |")
    return "\n".join(out)

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]

def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        out.append(f"### {d.get('Kernel Name','?')}")
        out.append("| metric | unit | value |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                out.append(f"| {k} | {units[hdr.index(k)]} | {d[k]} |")
    return "\n".join(out)

if __name__ == "__main__":
    kind, src, dst, title = sys.argv[1:5]
    body = launches(src) if kind == "launches" else full(src)
    open(dst, "w").write(f"# {title}\n\n{body}\n")
    print(open(dst).read()[:3000])
