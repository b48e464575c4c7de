"""Variant of tools/c4_filter_sim.py: group words plus a per-column extension
code ("+extE": E bits per column; the column's band widens by t buckets on
both sides when its own extremes reach that far), the shared-memory budget
being 200 KB (g5y8+ext1 = 64 KB of words + 128 KB of bits fits; +ext2 does
not).  usage: python tools/c4_filter_ext_sim.py 1e9 g4y8,g5y8+ext1,...
"""
import sys, time, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle
p = 1 << 20
N = int(float(sys.argv[1])); variants = sys.argv[2].split(',')
EMPTY = np.iinfo(np.int32).max
def words(lo, hi, gshift, hbits):
    ng = p >> gshift
    l = lo.reshape(ng, -1); h = hi.reshape(ng, -1)
    empty = (l > h).any(axis=1)
    maxlo = l.max(axis=1).astype(np.int64); minhi = h.min(axis=1).astype(np.int64)
    ys = 0
    while ((p - 1) >> ys) > (1 << hbits) - 1: ys += 1
    q = 1 << ys
    a = maxlo - 1
    fa = np.where(a <= 0, 0, (a + q - 1) // q)
    fb = np.where(minhi >= 0, minhi // q - 1, -1)
    fb = np.minimum(fb, (1 << hbits) - 1)
    never = empty | (fa > fb)
    fa = np.where(never, 1, fa); fb = np.where(never, 0, fb)
    return fa, fb, ys, never
def run(v):
    parts = v.split('+')
    g, yb = parts[0][1:].split('y'); gshift, hbits = int(g), int(yb)
    ext = int(parts[1][3:]) if len(parts) > 1 else 0
    lo = np.full(p, EMPTY, np.int32); hi = np.full(p, -1, np.int32)
    bounds = [0, N >> 6]
    while bounds[-1] < N: bounds.append(min(N, 2 * bounds[-1]))
    res = []
    for k in range(len(bounds) - 1):
        a, b = bounds[k], bounds[k + 1]
        if k:
            fa, fb, ys, never = words(lo, hi, gshift, hbits)
            q = 1 << ys
            gcol = np.arange(p) >> gshift
            fac = fa[gcol]; fbc = fb[gcol]
            e = np.zeros(p, np.int64)
            if ext:
                for t in range(1, (1 << ext)):
                    ok = (~never[gcol]) & (fac - t >= 0) & (lo.astype(np.int64) <= (fac - t) * q + 1) & (hi.astype(np.int64) >= (fbc + t + 1) * q)
                    e = np.where(ok, t, e)
            lo_b = fac - e; hi_b = fbc + e
        m_tot = 0
        for c0 in range(a, b, 1 << 24):
            c1 = min(b, c0 + (1 << 24))
            xy = oracle.generate(4, 4, p, c1 - c0, offset=c0)
            s = xy[:, 0].astype(np.int64) - 1; y = xy[:, 1].astype(np.int64)
            if k == 0:
                m = np.ones(len(s), bool)
            else:
                u = (y - 1) >> ys
                m = ~((u >= lo_b[s]) & (u <= hi_b[s]))
            ms = s[m]; my = y[m].astype(np.int32)
            m_tot += len(ms)
            np.minimum.at(lo, ms, my); np.maximum.at(hi, ms, my)
        res.append(m_tot)
    return res
for v in variants:
    t = time.time(); r = run(v)
    print(v, "total %.1f M" % (sum(r) / 1e6), [round(x / 1e6, 2) for x in r], "%.0fs" % (time.time() - t))
