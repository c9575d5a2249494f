"""Summarise ncu exports into profiles/ (committed evidence).

usage: python tools/summarize_ncu.py <launches.csv> <top_raw.csv> <out.md> [traffic.json]
  launches.csv : `ncu --metrics gpu__time_duration.sum --csv --log-file` output
  top_raw.csv  : `ncu -i <rep> --page raw --csv` of a --set full capture
"""
import csv
import io
import json
import re
import sys
from collections import defaultdict


def read_csv(path):
    txt = open(path, errors="replace").read()
    start = txt.find('"ID"')
    return list(csv.reader(io.StringIO(txt[start:])))


def base_name(k):
    k = re.sub(r"\(.*", "", k)
    k = k.replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return re.sub(r"^.*::", "", k)


def launches(path):
    rows = read_csv(path)
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        name = base_name(r[ki])
        if name.startswith("k_mul_peak"):  # the peak micro-benchmark, not part of a proof
            continue
        a = agg[name]
        a[0] += 1
        a[1] += ms
    return agg


def top(path):
    rows = read_csv(path)
    hdr = rows[0]
    want = ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
    units = rows[1] if len(rows) > 1 else []
    out = []
    for r in rows[2:]:
        d = {"kernel": base_name(r[hdr.index("Kernel Name")])}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                d[w] = (r[i], units[i] if i < len(units) else "")
        out.append(d)
    return out


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


def main():
    lpath, tpath, opath = sys.argv[1:4]
    tjson = sys.argv[4] if len(sys.argv) > 4 else None
    agg = launches(lpath)
    total = sum(v[1] for v in agg.values())
    lines = ["# ncu summary", "", f"Launch list: `{lpath}` (ncu --metrics gpu__time_duration.sum --clock-control none;",
             "cold-cache, serialised launches: compare shares, not absolutes).", "",
             "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.2f} | {100 * ms / total:.1f}% |")
    lines += ["", f"Total kernel time: {total:.2f} ms", "", "## Top kernels (--set full)", ""]
    traffic = []
    for d in top(tpath):
        lines.append(f"### `{d['kernel']}`")
        for k, vu in d.items():
            if k == "kernel":
                continue
            lines.append(f"- {k}: {vu[0]} {vu[1]}")
        if d["kernel"].startswith("k_round<") and "dram__bytes_read.sum" in d:
            rb = to_bytes(*d["dram__bytes_read.sum"])
            wb = to_bytes(*d["dram__bytes_write.sum"])
            traffic.append({"grid": d.get("launch__grid_size", ("", ""))[0], "dram_bytes": rb + wb})
        lines.append("")
    open(opath, "w").write("\n".join(lines) + "\n")
    if tjson and traffic:
        json.dump({"kernel": "k_round", "source": tpath, "launches": traffic,
                   "dram_bytes_per_launch": sum(t["dram_bytes"] for t in traffic) / len(traffic)},
                  open(tjson, "w"), indent=1)
    print(f"wrote {opath}")


if __name__ == "__main__":
    main()
