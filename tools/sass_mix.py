"""Per-kernel counts of the sm_100a-specific / warp-level SASS instructions in libdexel.so
(static counts from cuobjdump -sass): FADD2 (packed f32x2 add), REDUX (warp min), VOTE (ballot),
LDGSTS/LDGDEPBAR (cp.async), FLO/BREV/POPC (window bit scans), FMNMX / VIMNMX (min/max).
usage: python tools/sass_mix.py [libdexel.so]"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1804_08968_b200/libdexel.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["FADD2", "REDUX", "VOTE", "LDGSTS", "LDGDEPBAR", "FLO", "BREV", "POPC", "SHF", "FMNMX", "VIMNMX", "STG", "LDG"]
cur, cnt = None, collections.defaultdict(collections.Counter)
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        cnt[cur][m.group(2)] += 1
print("kernel | " + " | ".join(keys) + " | total")
for f in sorted(cnt):
    if "kernel" not in f:
        continue
    c = cnt[f]
    name = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip().split("(")[0]
    print(name + " | " + " | ".join(str(c[k]) for k in keys) + f" | {sum(c.values())}")
