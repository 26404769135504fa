"""Wall-clock and per-kernel time of one op (debug helper).
usage: python tools/time_op.py C4 dilate 1 [iters]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dexelgen as G  # noqa: E402
import paper_1804_08968_b200 as dx  # noqa: E402

cfg, op, r = sys.argv[1], sys.argv[2], float(sys.argv[3])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 5
host = G.config(cfg)
src = dx.Grid.from_host(host)
dst = dx.Grid.like(src)


def run():
    if op == "shell":
        dx.dexel_shell(src, r, r, dst)
    else:
        getattr(dx, "dexel_" + op)(src, r, dst)


for _ in range(3):
    run()
dst.sync()
for timing in (False, True):
    dx.set_timing(timing)
    t = time.perf_counter()
    for _ in range(iters):
        run()
    dst.sync()
    dt = (time.perf_counter() - t) / iters
    st = dst.stats()
    print(f"{cfg} {op} r={r} timing={timing}: wall {1e3*dt:.2f} ms/op; kernels "
          f"{sum(st['kernel_ms'].values()):.2f} ms {({k: round(v, 2) for k, v in st['kernel_ms'].items()})}")
print(f"  n_in={st['n_in']} n_mid={st['n_mid']} n_lev={st['n_lev']} n_out={st['n_out']} launches={st['launches']} "
      f"capacities={st['capacities']}")
