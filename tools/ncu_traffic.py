"""Sum ncu --set full captures per kernel kind (one op's launches) -> profiles/traffic.json.
usage: python tools/ncu_traffic.py report.ncu-rep|raw.csv KEY_PREFIX [traffic.json]   (KEY_PREFIX e.g. C5:shell:16.0)
Kernel kinds follow bench.py: p1_kernel -> pass1, levels_kernel -> levels, pass2s -> pass2."""
import csv
import json
import os
import subprocess
import sys

rep, prefix = sys.argv[1], sys.argv[2]
out = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
kinds = {"p1g_kernel": "pass1", "p1s_kernel": "pass1", "levels_kernel": "levels", "pass2s_kernel": "pass2"}
acc = {}
for r in rows[2:]:
    name = r[ix["Kernel Name"]]
    kind = next((v for k, v in kinds.items() if k in name), None)
    if kind is None:
        continue
    try:
        rd = float(r[ix["dram__bytes_read.sum"]]) * scale[units[ix["dram__bytes_read.sum"]]]
        wr = float(r[ix["dram__bytes_write.sum"]]) * scale[units[ix["dram__bytes_write.sum"]]]
    except ValueError:
        continue
    if rd != rd or wr != wr:   # nan rows (second pass of a replayed range)
        continue
    a = acc.setdefault(kind, {"read": 0.0, "write": 0.0, "launches": 0})
    a["read"] += rd
    a["write"] += wr
    a["launches"] += 1
path = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                           "profiles", "traffic.json")
tj = json.load(open(path)) if os.path.exists(path) else {}
for kind, a in acc.items():
    tj[f"{prefix}:{kind}"] = a["read"] + a["write"]
    tj[f"{prefix}:{kind}:detail"] = a
json.dump(tj, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(acc, indent=1))
