"""Markdown table of a bench matrix (jsonl of bench.py lines) for BASELINE.md section 3 / DESIGN.md."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
print("| config | op | r | ms/op | columns/s | e2e columns/s | dominant kernel | its GB/s (frac of measured peak) "
      "| DRAM traffic / algorithmic | oracle columns/s (cores) | GPU / oracle |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c = d["config"]
    rf = d.get("roofline") or {}
    cpu = d.get("cpu_baseline") or {}
    e2e = d.get("e2e") or {}
    tr = rf.get("traffic")
    ratio = f"{tr / rf['algorithmic_bytes_per_step']:.2f}" if tr and rf.get("algorithmic_bytes_per_step") else "-"
    print(f"| {c['workload'].split()[0]} | {c['op']} | {c['r']:g} | {d['ms_per_step']:.3f} | {d['value']:.3g} | "
          f"{e2e.get('value', 0):.3g} | {rf.get('kernel', '-')} | {rf.get('achieved', 0):.0f} ({rf.get('frac', 0):.3f}) | "
          f"{ratio} | {cpu.get('value', 0):.3g} ({cpu.get('cores', '-')}) | "
          f"{d['value'] / cpu['value'] if cpu.get('value') else 0:.0f}x |")
