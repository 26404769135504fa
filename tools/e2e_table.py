"""e2e summary of bench lines: python tools/e2e_table.py FILE.jsonl"""
import json
import sys

print("| workload | device ms/op | e2e api | e2e ms/step | e2e columns/s | serial e2e ms/step | serial columns/s |")
print("|---|---|---|---|---|---|---|")
for l in open(sys.argv[1]):
    l = l.strip()
    if not l.startswith("{"):
        continue
    d = json.loads(l)
    e = d.get("e2e") or {}
    s = e.get("serial") or {}
    print(f"| {d['config']['workload']} | {d['ms_per_step']:.2f} | {e.get('api', '-')} | {e.get('ms_per_step', 0):.2f} | "
          f"{e.get('value', 0):.3g} | {s.get('ms_per_step', 0):.2f} | {s.get('value', 0):.3g} |")
