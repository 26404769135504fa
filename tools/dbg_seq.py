"""debug helper: a sequence of C4 dilate ops in one process (as the parity tests run them)"""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(90, exit=True)
import dexelgen as G
import paper_1804_08968_b200 as dx
host = G.config("C4")
for r in [float(x) for x in sys.argv[1:]]:
    t = time.time()
    src = dx.Grid.from_host(host)
    dst = dx.Grid.like(src)
    dx.dexel_dilate(src, r, dst)
    off, ep = dst.download()
    print(r, "ok", round(time.time() - t, 2), dst.stats()["capacities"], flush=True)
    src.close(); dst.close()
