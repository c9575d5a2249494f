"""Brief per-launch summary of an .ncu-rep: duration, DRAM bytes, issue %, pipes, top stalls."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
keys = {"dur_us": "gpu__time_duration.sum", "regs": "launch__registers_per_thread",
        "issue%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "alu%": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "fma%": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "inst": "smsp__inst_executed.sum", "dram_rd": "dram__bytes_read.sum", "dram_wr": "dram__bytes_write.sum",
        "bank_conf": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"}
for j, row in enumerate(r[2:]):
    out = {"kernel": row[h.index("Kernel Name")][:60]}
    for k, m in keys.items():
        if m in h:
            out[k] = row[h.index(m)]
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(row[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    out["stalls"] = ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:6])
    print(out)
