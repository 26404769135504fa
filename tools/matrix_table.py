"""Markdown table of a bench matrix (jsonl of bench.py lines) for BASELINE.md section 3 / DESIGN.md.
usage: python tools/matrix_table.py MATRIX.jsonl [PARITY.json]
PARITY.json: the GPU tests' parity report (DEXEL_PARITY_REPORT), keyed "<cfg> <op> r=<r>"."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
par = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else {}
print("| config | op | r | GPUs | ms/op | columns/s | e2e columns/s | dominant kernel | its GB/s (frac of measured peak) "
      "| DRAM traffic / algorithmic | oracle columns/s (cores) | parity: max error, count mismatches (columns compared) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c = d["config"]
    rf = d.get("roofline") or {}
    cpu = d.get("cpu_baseline") or {}
    e2e = d.get("e2e") or {}
    tr = rf.get("traffic")
    ratio = f"{tr / rf['algorithmic_bytes_per_step']:.2f}" if tr and rf.get("algorithmic_bytes_per_step") else "-"
    cfg = c["workload"].split()[0]
    p = par.get(f"{cfg} {c['op']} r={float(c['r'])}")
    ptxt = f"{p['max_err']:.1e}, {p['count_mismatch']} ({p['columns']})" if p else "-"
    print(f"| {cfg} | {c['op']} | {c['r']:g} | {d.get('n_gpus', 1)} | {d['ms_per_step']:.3f} | {d['value']:.3g} | "
          f"{e2e.get('value', 0):.3g} | {rf.get('kernel', '-')} | {rf.get('achieved', 0):.0f} ({rf.get('frac', 0):.3f}) | "
          f"{ratio} | {cpu.get('value', 0):.3g} ({cpu.get('cores', '-')}) | {ptxt} |")
