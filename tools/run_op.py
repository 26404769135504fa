"""Run one op on one config a few times (for ncu / compute-sanitizer targeting).
usage: python tools/run_op.py C4 dilate 16 [iters]
With PROFILE_LAST=1 the CUDA profiler is started just before the last op (run ncu with
--profile-from-start off to capture the steady-state op only: capacity hints already grown)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dexelgen as G  # noqa: E402
import paper_1804_08968_b200 as dx  # noqa: E402

cfg, op, r = sys.argv[1], sys.argv[2], float(sys.argv[3])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 2
last = os.environ.get("PROFILE_LAST") == "1"
cudart = None
if last:
    import torch
    cudart = torch.cuda.cudart()
host = G.config(cfg)
src = dx.Grid.from_host(host)
dst = dx.Grid.like(src)
for it in range(iters):
    if last and it == iters - 1:
        dst.sync()
        cudart.cudaProfilerStart()
    if op == "shell":
        dx.dexel_shell(src, r, r, dst)
    else:
        getattr(dx, "dexel_" + op)(src, r, dst)
dst.sync()
if last:
    cudart.cudaProfilerStop()
print(cfg, op, r, dst.stats())
