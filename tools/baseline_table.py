"""BASELINE.md section-3 table from a bench matrix (jsonl) and the GPU tests' parity report.
usage: python tools/baseline_table.py MATRIX.jsonl PARITY.json"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
par = json.load(open(sys.argv[2]))
print("| config | op | r | GPUs | GPU columns/s (ms/op) | e2e columns/s | dominant kernel: algorithmic GB/s (fraction of the measured 6456 GB/s) "
      "| oracle columns/s | host cores | parity (max error, count mismatches, columns compared) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c = d["config"]
    rf = d.get("roofline") or {}
    cpu = d.get("cpu_baseline") or {}
    cfg = c["workload"].split()[0]
    p = par.get(f"{cfg} {c['op']} r={float(c['r'])}")
    ptxt = f"{p['max_err']:.1e}, {p['count_mismatch']}, {p['columns']}" if p else "-"
    lb = " (launch-bound)" if cfg in ("C1", "C2") else ""
    print(f"| {cfg} {c['grid']} | {c['op']} | {c['r']:g} | {d.get('n_gpus', 1)} | {d['value']:.3g} ({d['ms_per_step']:.3f}) | "
          f"{(d.get('e2e') or {}).get('value', 0):.3g} | {rf.get('kernel', '-')}: {rf.get('achieved', 0):.0f} ({rf.get('frac', 0):.3f}){lb} | "
          f"{cpu.get('value', 0):.3g} | {cpu.get('cores', '-')} | {ptxt} |")
