"""One-line-per-launch summary of an ncu --set full report (for profiles/)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}
cols = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "simt"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "inst")]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
print("# " + sys.argv[2] if len(sys.argv) > 2 else "#")
print("kernel | " + " | ".join(f"{n} [{units[ix[m]]}]" for m, n in cols if m in ix) + " | top stalls (cycles per issue)")
for r in rows[2:]:
    vals = [r[ix[m]] for m, n in cols if m in ix]
    if any(v in ("nan", "-nan") for v in vals):
        continue
    st = sorted(((float(r[ix[h]]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                 for h in stalls if r[ix[h]] not in ("nan", "-nan")), reverse=True)[:4]
    print(r[ix["Kernel Name"]].split("(")[0] + " | " + " | ".join(vals) + " | " + ", ".join(f"{n} {v:.2f}" for v, n in st))
