"""Host simulation of K1's column-group filter on BASELINE.json config 4
(n points of the C4 stream, p = 2^20): per phase of the doubling schedule
(warm-up n/64 with an empty table, then [d, 2d) against a snapshot of L at d),
how many points miss the filter -- i.e. touch L2 -- for group sizes 2^g
columns and H-bit word halves ("g4y8" = the device's 16-column groups with
8-bit halves), and for an exact per-column snapshot ("exact", which does not
fit shared memory at p = 2^20).  The device's filter words follow
k_filter_build's rule (reduce.cu); the miss counts match ncu's RED/read counts
per phase (profiles/r02_ncu_full_summary.md).

usage: python tools/c4_filter_sim.py <n> <variant,...>    e.g. 1e9 g4y8,g4y12,g3y8,exact
"""
import sys, time, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle
p = 1 << 20
N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
variants = sys.argv[2].split(',') if len(sys.argv) > 2 else ['g4y12']
EMPTY_LO = np.iinfo(np.int32).max

def words(lo, hi, gshift, hbits):
    # group band per the k_filter_build rule, returns (fa, fb) int64 arrays with fb<fa meaning never
    ng = p >> gshift
    l = lo.reshape(ng, -1); h = hi.reshape(ng, -1)
    empty = (l > h).any(axis=1)
    maxlo = l.max(axis=1).astype(np.int64); minhi = h.min(axis=1).astype(np.int64)
    ys = 0
    while ((p - 1) >> ys) > (1 << hbits) - 1: ys += 1
    q = 1 << ys
    a = maxlo - 1
    fa = np.where(a <= 0, 0, (a + q - 1) // q)
    b = minhi - 1 + 1
    fb = np.where(b >= 0, b // q - 1, -1)
    fb = np.minimum(fb, (1 << hbits) - 1)
    never = empty | (fa > fb)
    fa = np.where(never, 1, fa); fb = np.where(never, 0, fb)
    return fa, fb, ys

def run(variant, chunks):
    if variant == 'exact':
        gshift, hbits = 0, 31
    else:
        g, yb = variant[1:].split('y'); gshift, hbits = int(g), int(yb)
    lo = np.full(p, EMPTY_LO, np.int32); hi = np.full(p, -1, np.int32)
    warm = N >> 6
    bounds = [0, warm]
    while bounds[-1] < N: bounds.append(min(N, 2 * bounds[-1]))
    res = []
    for k in range(len(bounds) - 1):
        a, b = bounds[k], bounds[k + 1]
        if k == 0:
            fa = fb = None
        else:
            if variant == 'exact':
                fa, fb = lo.astype(np.int64), hi.astype(np.int64); ys = 0
                never = lo > hi
                fa = np.where(never, 1, fa); fb = np.where(never, 0, fb)
            else:
                fa, fb, ys = words(lo, hi, gshift, hbits)
        miss_tot = 0; upd = 0
        for c0 in range(a, b, 1 << 24):
            c1 = min(b, c0 + (1 << 24))
            xy = chunks(c0, c1)
            s = xy[:, 0].astype(np.int64) - 1; y = xy[:, 1].astype(np.int64)
            if fa is None:
                m = np.ones(len(s), bool)
            else:
                gi = s >> gshift
                u = (y - 1) >> ys if variant != 'exact' else y
                m = ~((u >= fa[gi]) & (u <= fb[gi]))
            ms = s[m]; my = y[m]
            miss_tot += len(ms)
            before_lo = lo[ms]; before_hi = hi[ms]
            upd += int(((my < before_lo) | (my > before_hi)).sum())
            np.minimum.at(lo, ms, my.astype(np.int32)); np.maximum.at(hi, ms, my.astype(np.int32))
        res.append((a, b, miss_tot, upd))
    return res

cache = {}
def chunks(a, b):
    key = (a, b)
    if key not in cache:
        cache[key] = oracle.generate(4, 4, p, b - a, offset=a)
    return cache[key]

for v in variants:
    t = time.time()
    r = run(v, chunks)
    tot = sum(x[2] for x in r)
    print(f"{v}: total misses {tot/1e6:.1f} M  ({time.time()-t:.0f}s)")
    for a, b, m, u in r:
        print(f"   [{a/N:.4f},{b/N:.4f})  n={(b-a)/1e6:7.1f}M  misses {m/1e6:6.2f}M ({m/(b-a)*100:5.1f}%)  first-seen-updates-est {u/1e6:5.2f}M")
