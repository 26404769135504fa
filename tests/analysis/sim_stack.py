"""Analysis script (not a test): how often the forward stack sweep of levels_kernel pops an already-written component, on the oracle's P1 pieces of sampled rows (DESIGN.md levels_kernel).
usage: python tests/analysis/sim_stack.py C5 16 [complement]"""
import sys, math, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))))
import dexelgen as G, oracle as O
cfg = sys.argv[1]; r = float(sys.argv[2]); comp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g = G.config(cfg)
R = int(r)
rows = [g.ny // 2 + d for d in range(0, 4)]
cols = np.array([j * g.nx + i for j in rows for i in range(0, g.nx, 7)], np.int64)
p = O.pass1(g, r, complement=bool(comp), cols=cols)
pairs = pushes = pops = ext = uf = ur = lk = 0
maxdepth = 0
for t in range(len(cols)):
    z = p.column(t); k = p.kappa(t)
    for lev in range(R + 1):
        top = None; stack = []
        for (lo, hi), kap in zip(z, k):
            w = r * r - (int(kap) ** 2 + lev * lev)
            if w < 0: continue
            h = math.sqrt(w); s, e = lo - h, hi + h
            pairs += 1
            if top is None: top = [s, e]; continue
            if s > top[1]:
                stack.append(top); top = [s, e]; pushes += 1
            else:
                top = [min(top[0], s), max(top[1], e)]
                d = 0
                while stack and stack[-1][1] >= top[0]:
                    top[0] = min(top[0], stack[-1][0]); stack.pop(); pops += 1; d += 1
                maxdepth = max(maxdepth, d)
        lk += len(stack) + (top is not None)
print(cfg, r, 'comp', comp, 'cols', len(cols), 'pieces/col %.1f' % (len(p.k) / len(cols)),
      'valid pairs/col %.1f' % (pairs / len(cols)), 'pushes/col %.1f' % (pushes / len(cols)),
      'deep pops/col %.2f' % (pops / len(cols)), 'maxdepth', maxdepth, '|L| per col %.1f' % (lk / len(cols)))
