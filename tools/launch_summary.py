"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file).
usage: python tools/launch_summary.py launches.csv "header line" > profiles/<name>.txt"""
import csv
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot, cnt = {}, {}
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).strip()
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    ms = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
    tot[name] = tot.get(name, 0.0) + ms
    cnt[name] = cnt.get(name, 0) + 1
s = sum(tot.values()) or 1.0
print("# " + (sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]))
print("# per-kernel totals over all launches of the run (warmup + timed steps); cold-cache, serialised: compare shares")
print(f"{'kernel':<40} {'launches':>9} {'total_ms':>10} {'share':>6}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:<40} {cnt[k]:>9} {tot[k]:>10.2f} {100 * tot[k] / s:>5.1f}%")
