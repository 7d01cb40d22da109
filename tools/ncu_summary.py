"""Summarise ncu artefacts into profiles/ (run here, after gpurun brought them back).

    python tools/ncu_summary.py <prof.ncu-rep> <launches.csv> <out_prefix>

Writes <out_prefix>_summary.md (top-kernel metrics + launch-share table) and
profiles/tc_matcher_traffic.json (DRAM bytes per launch of k_match_tc, read by
bench.py's roofline `traffic`).
"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__block_size",
    "launch__grid_size",
    "sm__cycles_elapsed.avg.per_second",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, n in enumerate(hdr):
            if n in WANT or n == "Kernel Name":
                d[n] = (r[i], units[i])
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg, tot = {}, 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name] = agg.get(name, 0.0) + v
        tot += v
    return agg, tot


def main():
    rep, lcsv, prefix = sys.argv[1:4]
    lines = [f"# ncu summary ({os.path.basename(rep)}, {os.path.basename(lcsv)})", ""]
    ms = raw_metrics(rep)
    for d in ms:
        name = d.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in WANT:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        lines.append("")
        if "k_match_tc" in name and "dram__bytes_read.sum" in d and "cfg3" in os.path.basename(rep):
            def to_bytes(v, u):
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            tr = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
            with open(os.path.join(os.path.dirname(prefix) or ".", "tc_matcher_traffic.json"), "w") as f:
                json.dump({"dram_bytes_per_launch": tr, "source": os.path.basename(rep)}, f)
        for kname in ("k_pool", "k_domrows"):
            if kname in name and "dram__bytes_read.sum" in d and "cfg3" in os.path.basename(rep):
                tr = sum(float(d[m][0].replace(",", "")) *
                         {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d[m][1], 1)
                         for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                path = os.path.join(os.path.dirname(prefix) or ".", "k1_traffic.json")
                cur = json.load(open(path)) if os.path.exists(path) else {}
                cur[kname] = tr
                cur["source"] = os.path.basename(rep)
                with open(path, "w") as f:
                    json.dump(cur, f)
    agg, tot = launches(lcsv)
    lines += ["## launch list (ncu gpu__time_duration, serialised, cold caches)", "",
              "| kernel | time (us) | share |", "|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"| {k[:80]} | {v:.1f} | {100 * v / tot:.2f}% |")
    lines.append(f"| total | {tot:.1f} | 100% |")
    with open(prefix + "_summary.md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
