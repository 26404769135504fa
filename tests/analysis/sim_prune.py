"""Analysis script (not a test): pieces per column left by the adjacent-pair capsule-domination filter vs. an all-pairs test vs. greedy level-set redundancy, on the oracle's P1 pieces of sampled rows (DESIGN.md p1_kernel).
usage: python tests/analysis/sim_prune.py C5 16 [complement]"""
import sys, math, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))))
import dexelgen as G, oracle as O
cfg = sys.argv[1]; r = float(sys.argv[2]); comp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g = G.config(cfg); R = int(r)
H0 = [math.sqrt(max(0.0, r*r - a*a)) for a in range(R + 1)]
def h(k, lev):
    w = r*r - (k*k + lev*lev); return math.sqrt(w) if w >= 0 else None
rows = [g.ny // 2 + d for d in range(0, 3)]
cols = np.array([j * g.nx + i for j in rows for i in range(0, g.nx, 11)], np.int64)
p = O.pass1(g, r, complement=bool(comp), cols=cols)
def dom(q, pp):   # q dominates pp
    (lq, hq, kq), (lp, hp, kp) = q, pp
    return kq <= kp and max(lq - lp, hp - hq) <= H0[kq] - H0[kp] - 1e-6 * (1 + abs(H0[kq] - H0[kp]))
def levels(ps):
    out = []
    for lev in range(R + 1):
        iv = sorted((lo - h(k, lev), hi + h(k, lev)) for lo, hi, k in ps if h(k, lev) is not None)
        m = []
        for a, b in iv:
            if m and a <= m[-1][1]: m[-1][1] = max(m[-1][1], b)
            else: m.append([a, b])
        out.append(m)
    return out
tot_un = tot_adj = tot_any = tot_red = 0
for t in range(len(cols)):
    z = p.column(t); k = p.kappa(t)
    ps = [(float(a), float(b), int(c)) for (a, b), c in zip(z, k)]
    tot_un += len(ps)
    # adjacent pending filter (GPU rule)
    kept = []; pend = None
    for n in ps:
        if pend is None: pend = n; continue
        if dom(pend, n): continue
        if not dom(n, pend): kept.append(pend)
        pend = n
    if pend is not None: kept.append(pend)
    tot_adj += len(kept)
    # dominated by any other kept piece
    rem = [x for i, x in enumerate(kept) if not any(j != i and dom(y, x) for j, y in enumerate(kept))]
    tot_any += len(rem)
    # greedy redundancy: drop a piece if the level sets stay the same (limited to sample)
    if t % 8 == 0:
        L0 = levels(rem); cur = list(rem); red = 0
        for x in list(rem):
            trial = [y for y in cur if y is not x]
            if levels(trial) == L0: cur = trial; red += 1
        tot_red += red * 8
n = len(cols)
print(cfg, r, 'comp', comp, 'unpruned/col %.1f' % (tot_un / n), 'adjacent-filter %.1f' % (tot_adj / n),
      'any-pair %.1f' % (tot_any / n), 'further redundant (est) %.1f' % (tot_red / n))
