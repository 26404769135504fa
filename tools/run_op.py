"""Run one op on one config a few times (for ncu / compute-sanitizer targeting).
usage: python tools/run_op.py C4 dilate 16 [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dexelgen as G  # noqa: E402
import paper_1804_08968_b200 as dx  # noqa: E402

cfg, op, r = sys.argv[1], sys.argv[2], float(sys.argv[3])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 2
host = G.config(cfg)
src = dx.Grid.from_host(host)
dst = dx.Grid.like(src)
for _ in range(iters):
    if op == "shell":
        dx.dexel_shell(src, r, r, dst)
    else:
        getattr(dx, "dexel_" + op)(src, r, dst)
dst.sync()
print(cfg, op, r, dst.stats())
