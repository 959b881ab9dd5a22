"""Per-kernel summary of an ncu --set full report (raw page): duration, FP64 pipe, issue active, warps
active, registers, DRAM bytes (total and per element), the largest stall reasons per issue.
usage: python tools/ncu_summary.py <report.ncu-rep> [elements]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nel = int(sys.argv[2]) if len(sys.argv) > 2 else 10368
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
SC = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def val(r, name):
    i = col[name]
    return float(r[i].replace(",", "")) * SC.get(units[i], 1.0)


print("| kernel | ncu duration (ms) | FP64 pipe | issue active | warps active | regs | DRAM bytes / element | largest stalls (warps per issue) |")
print("|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    st = {h.split("issue_stalled_")[1].split("_per_issue")[0]: float(r[i]) for h, i in col.items()
          if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio") and "selected" not in h}
    top = ", ".join("%s %.2f" % kv for kv in sorted(st.items(), key=lambda kv: -kv[1])[:5])
    dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    print("| `%s` | %.3f | %.1f %% | %.1f %% | %.1f %% | %d | %.0f | %s |" % (
        r[col["Kernel Name"]].replace("void ", "").split("(")[0], val(r, "gpu__time_duration.sum"),
        val(r, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
        val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        int(float(r[col["launch__registers_per_thread"]])), dram / nel, top))
