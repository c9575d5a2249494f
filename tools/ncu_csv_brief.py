"""Per-launch summary of ncu --page raw --csv exports (.csv or .csv.gz):
duration, DRAM bytes and GB/s, issue and pipe utilisation, top stalls.
usage: python tools/ncu_csv_brief.py file.csv[.gz] ..."""
import csv
import gzip
import io
import sys

KEYS = {"dur_us": "gpu__time_duration.sum", "regs": "launch__registers_per_thread", "grid": "launch__grid_size",
        "issue%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "alu%": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "fma%": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram_rd_MB": "dram__bytes_read.sum", "dram_wr_MB": "dram__bytes_write.sum"}


def rows(path):
    raw = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read().splitlines()
    start = next(i for i, l in enumerate(raw) if l.startswith('"ID"'))
    r = list(csv.reader(raw[start:]))
    return r[0], r[1], r[2:]


for path in sys.argv[1:]:
    h, units, data = rows(path)
    for row in data:
        out = {"kernel": row[h.index("Kernel Name")].split("(")[0].replace("void unnamed>::", "")[:48]}
        for k, m in KEYS.items():
            if m in h:
                v = row[h.index(m)]
                u = units[h.index(m)]
                try:
                    x = float(v)
                    if k.endswith("_MB") and u == "Gbyte":
                        x *= 1e3
                    elif k.endswith("_MB") and u == "Kbyte":
                        x /= 1e3
                    elif k == "dur_us" and u == "ms":
                        x *= 1e3
                    elif k == "dur_us" and u == "ns":
                        x /= 1e3
                    out[k] = round(x, 2)
                except ValueError:
                    out[k] = v
        if "dur_us" in out and "dram_rd_MB" in out:
            out["dram_GBps"] = round((out["dram_rd_MB"] + out.get("dram_wr_MB", 0)) / out["dur_us"] * 1e3, 1)
        st = []
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(row[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        out["top_stalls"] = ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:4])
        print(out)
