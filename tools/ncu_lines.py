"""Per-source-line warp-stall samples and instruction counts from an ncu report.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, h, out = "", None, []
for r in csv.reader(txt.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]; h = None; continue
    if r[0] == "Line No":
        h = r; continue
    if h and len(r) == len(h) and r[0]:
        try:
            s = int(r[4] or 0); ie = int(r[7] or 0)
        except ValueError:
            continue
        out.append((s, ie, f"{fn}:{r[0]}", r[1].strip()[:90]))
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"samples {tot} instructions {ti}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{100*o[0]/tot:6.2f}% {100*o[1]/ti:6.2f}%  {o[2]:<18} {o[3]}")

if len(sys.argv) > 3:      # stall breakdown of the given source lines, e.g. levels.cuh:262,levels.cuh:188
    want = set(sys.argv[3].split(","))
    names = ["barrier", "branch", "dispatch", "drain", "lg", "long_sb", "math", "membar", "mio", "misc",
             "no_inst", "not_sel", "selected", "short_sb", "sleep", "tex", "wait"]
    fn, h = "", None
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fn = r[1].split("/")[-1]; h = None; continue
        if r[0] == "Line No":
            h = r; continue
        if h and len(r) == len(h) and r[0] and f"{fn}:{r[0]}" in want:
            v = [int(x or 0) for x in r[31:48]]
            tot_l = sum(v) or 1
            print(f"{fn}:{r[0]:<5}", " ".join(f"{n}={100*x/tot_l:.0f}%" for n, x in zip(names, v) if x > 0.03 * tot_l))
