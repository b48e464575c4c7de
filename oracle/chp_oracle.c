/*
 * chp_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see chp_oracle.h).  Plain C11; exact integer
 * arithmetic throughout.  Citations are relative to /root/reference/proj.
 */
#include "chp_oracle.h"

#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <pthread.h>

typedef __int128 i128;

/* ---------------------------------------------------------------- digest */

uint64_t or_fnv1a64(const void* data, size_t len) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

/* ------------------------------------------------------------- generator */

/* std::mt19937_64 (the standard's parameter set). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
                   (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (g->mt[k] & upper) | (g->mt[(k + 1) % 312] & lower);
            uint64_t v = g->mt[(k + 156) % 312] ^ (y >> 1);
            if (y & 1) v ^= 0xB5026F5AA96619E9ull;
            g->mt[k] = v;
        }
        g->idx = 0;
    }
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

/* libstdc++ (GCC 13) uniform_int_distribution<int64_t>(a,b) with a 64-bit
 * engine: Lemire's nearly-divisionless method over a 128-bit product
 * (bits/uniform_int_dist.h, _S_nd). */
static int64_t uniform_int(mt64* g, int64_t a, int64_t b) {
    const uint64_t range = (uint64_t)(b - a) + 1u;
    unsigned __int128 prod = (unsigned __int128)mt64_next(g) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
        const uint64_t threshold = (0u - range) % range;
        while (low < threshold) {
            prod = (unsigned __int128)mt64_next(g) * range;
            low = (uint64_t)prod;
        }
    }
    return a + (int64_t)(uint64_t)(prod >> 64);
}

void or_gen_uniform_box(uint64_t n, int64_t p, uint64_t seed, int32_t* xy) {
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    for (uint64_t i = 0; i < n; ++i) {
        /* x before y: pts.push_back({coord(rng), coord(rng)}) is evaluated
         * left to right in a braced initializer (src/dataset.cpp:59). */
        xy[2 * i] = (int32_t)uniform_int(g, 1, p);
        xy[2 * i + 1] = (int32_t)uniform_int(g, 1, p);
    }
    free(g);
}

/* ------------------------------------------------------------ reduction */

static void occ_insert(uint64_t* occ, uint64_t i /* 1-based */) {
    /* bit_index_map(i, 64): block (i-1)>>6, position (i-1)&63
     * (include/chp/occupancy.hpp:46-49), insert at :70-74. */
    occ[(i - 1) >> 6] |= 1ull << ((i - 1) & 63);
}

void or_bucket(const int32_t* xy, uint64_t n, int64_t x_off, int32_t* lo,
               int32_t* hi, uint8_t* valid, uint64_t* occ) {
    for (uint64_t k = 0; k < n; ++k) {
        const int64_t x = (int64_t)xy[2 * k] - x_off;
        const int32_t y = xy[2 * k + 1];
        const int64_t s = x - 1;
        if (!valid[s]) {
            lo[s] = y;
            hi[s] = y;
            valid[s] = 1;
            if (occ) occ_insert(occ, (uint64_t)x);
        } else {
            if (y < lo[s]) lo[s] = y;
            if (y > hi[s]) hi[s] = y;
        }
    }
}

int or_reduce(const int32_t* xy, uint64_t n, int64_t width, int64_t q,
              int32_t* lo, int32_t* hi, uint8_t* valid, uint64_t* occ) {
    if (width < 1) return -1;
    for (uint64_t k = 0; k < n; ++k) {
        const int64_t x = xy[2 * k], y = xy[2 * k + 1];
        if (x < 1 || x > width || y < 1 || (q >= 0 && y > q)) return -1;
    }
    for (int64_t s = 0; s < width; ++s) {
        lo[s] = 0;   /* ColumnExtremes defaults, include/chp/reducer.hpp:19-25 */
        hi[s] = -1;
        valid[s] = 0;
    }
    if (occ) memset(occ, 0, (size_t)((width + 63) / 64) * sizeof(uint64_t));
    or_bucket(xy, n, 0, lo, hi, valid, occ);
    return 0;
}

/* SURVEY.md 8(c)'s chunked procedure for inputs beyond one reduce() call:
 * reduce() (src/reducer.cpp:69-79) per slice on `threads` host threads, each
 * into a private (lo, hi, valid), then the slot-by-slot merge of the
 * partials -- exact because min/max are associative and commutative, the
 * property tests/test_reducer.cpp:113-127 pins (reducing the survivors
 * again reproduces L).  Accumulates into the caller's arrays (initialise
 * them once with valid = 0); the validation of src/reducer.cpp:72-75 runs on
 * every point.  Returns 0, or -1 when the reference would throw. */
typedef struct {
    const int32_t* xy;
    uint64_t n;
    int64_t width, q;
    int32_t *lo, *hi;
    uint8_t* valid;
    int rc;
} fold_job;

static void* fold_worker(void* arg) {
    fold_job* j = (fold_job*)arg;
    j->rc = 0;
    for (uint64_t k = 0; k < j->n; ++k) {
        const int64_t x = j->xy[2 * k], y = j->xy[2 * k + 1];
        if (x < 1 || x > j->width || y < 1 || (j->q >= 0 && y > j->q)) {
            j->rc = -1;
            return NULL;
        }
    }
    for (int64_t s = 0; s < j->width; ++s) j->valid[s] = 0;
    or_bucket(j->xy, j->n, 0, j->lo, j->hi, j->valid, NULL);
    return NULL;
}

int or_reduce_accumulate_mt(const int32_t* xy, uint64_t n, int64_t width, int64_t q,
                            int threads, int32_t* lo, int32_t* hi, uint8_t* valid) {
    if (width < 1) return -1;
    if (threads < 1) threads = 1;
    if (threads > 64) threads = 64;
    if ((uint64_t)threads > n / 4096 + 1) threads = (int)(n / 4096 + 1);
    fold_job* jobs = (fold_job*)calloc((size_t)threads, sizeof(fold_job));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    int rc = 0;
    for (int t = 0; t < threads; ++t) {
        const uint64_t a = n * (uint64_t)t / (uint64_t)threads, b = n * (uint64_t)(t + 1) / (uint64_t)threads;
        jobs[t].xy = xy + 2 * a;
        jobs[t].n = b - a;
        jobs[t].width = width;
        jobs[t].q = q;
        jobs[t].lo = (int32_t*)malloc((size_t)width * 4);
        jobs[t].hi = (int32_t*)malloc((size_t)width * 4);
        jobs[t].valid = (uint8_t*)malloc((size_t)width);
        pthread_create(&tid[t], NULL, fold_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) {
        pthread_join(tid[t], NULL);
        if (jobs[t].rc) rc = -1;
    }
    for (int t = 0; t < threads && rc == 0; ++t) {
        const fold_job* j = &jobs[t];
        for (int64_t s = 0; s < width; ++s) {
            if (!j->valid[s]) continue;
            if (!valid[s]) {
                lo[s] = j->lo[s];
                hi[s] = j->hi[s];
                valid[s] = 1;
            } else {
                if (j->lo[s] < lo[s]) lo[s] = j->lo[s];
                if (j->hi[s] > hi[s]) hi[s] = j->hi[s];
            }
        }
    }
    for (int t = 0; t < threads; ++t) {
        free(jobs[t].lo);
        free(jobs[t].hi);
        free(jobs[t].valid);
    }
    free(jobs);
    free(tid);
    return rc;
}

/* The occupancy words of a merged (valid) array: Index::insert for every
 * valid slot (include/chp/occupancy.hpp:70-74). */
void or_occ_from_valid(int64_t width, const uint8_t* valid, uint64_t* occ) {
    memset(occ, 0, (size_t)((width + 63) / 64) * sizeof(uint64_t));
    for (int64_t s = 0; s < width; ++s)
        if (valid[s]) occ_insert(occ, (uint64_t)s + 1);
}

void or_L_pairs(int64_t width, const int32_t* lo, const int32_t* hi,
                const uint8_t* valid, int32_t* out) {
    for (int64_t s = 0; s < width; ++s) {
        out[2 * s] = valid[s] ? lo[s] : (int32_t)(width + 1);
        out[2 * s + 1] = valid[s] ? hi[s] : -1;
    }
}

size_t or_serialize(int64_t width, const int32_t* lo, const int32_t* hi,
                    const uint8_t* valid, char* buf, size_t cap) {
    size_t used = 0;
    char line[80];
    for (int64_t i = 1; i <= width; ++i) {
        int len;
        if (valid[i - 1])
            len = snprintf(line, sizeof line, "%lld %d %d\n", (long long)i,
                           lo[i - 1], hi[i - 1]);
        else
            len = snprintf(line, sizeof line, "%lld %lld -1\n", (long long)i,
                           (long long)(width + 1));
        if (buf && used + (size_t)len <= cap) memcpy(buf + used, line, (size_t)len);
        used += (size_t)len;
    }
    return used;
}

/* ------------------------------------------------------------ compaction */

/* Visit set bits in increasing order, one ctz per bit
 * (include/chp/occupancy.hpp:83-93). */
#define OCC_FOR_EACH(occ, width, I, BODY)                                   \
    do {                                                                    \
        const uint64_t nwords_ = (uint64_t)(((width) + 63) / 64);           \
        for (uint64_t b_ = 0; b_ < nwords_; ++b_) {                         \
            uint64_t w_ = (occ)[b_];                                        \
            while (w_) {                                                    \
                const int pos_ = __builtin_ctzll(w_);                       \
                w_ ^= 1ull << pos_;                                         \
                const uint64_t I = b_ * 64 + (uint64_t)pos_ + 1;            \
                BODY;                                                       \
            }                                                               \
        }                                                                   \
    } while (0)

int64_t or_valid_count(int64_t width, const int32_t* lo, const int32_t* hi,
                       const uint64_t* occ) {
    int64_t count = 0;
    OCC_FOR_EACH(occ, width, i, { count += lo[i - 1] == hi[i - 1] ? 1 : 2; });
    return count;
}

static void put_original(int32_t* out, int64_t k, int64_t slot, int64_t value,
                         int64_t major_off, int64_t minor_off, int swapped) {
    /* ExtremalArray::to_original, include/chp/reducer.hpp:46-50. */
    const int64_t major = slot + major_off, minor = value + minor_off;
    out[2 * k] = (int32_t)(swapped ? minor : major);
    out[2 * k + 1] = (int32_t)(swapped ? major : minor);
}

int64_t or_build_polyline(int64_t width, const int32_t* lo, const int32_t* hi,
                          const uint64_t* occ, int64_t major_off,
                          int64_t minor_off, int swapped, int32_t* chain) {
    int64_t k = 0;
    OCC_FOR_EACH(occ, width, i, {
        const int64_t slot = (int64_t)i;
        put_original(chain, k++, slot, lo[i - 1], major_off, minor_off, swapped);
        if (hi[i - 1] != lo[i - 1])
            put_original(chain, k++, slot, hi[i - 1], major_off, minor_off, swapped);
    });
    return k == 0 ? -1 : k;
}

int64_t or_ns_chain(int64_t width, const int32_t* lo, const int32_t* hi,
                    const uint64_t* occ, int64_t major_off, int32_t* chain) {
    int64_t k = 0;
    OCC_FOR_EACH(occ, width, i, {
        put_original(chain, k++, (int64_t)i, lo[i - 1], major_off, 0, 0);
    });
    for (int64_t i = width; i >= 1; --i) {
        const uint64_t b = (uint64_t)(i - 1);
        if (!((occ[b >> 6] >> (b & 63)) & 1)) continue;
        if (hi[i - 1] != lo[i - 1])
            put_original(chain, k++, i, hi[i - 1], major_off, 0, 0);
    }
    return k == 0 ? -1 : k;
}

/* ------------------------------------------------------------- geometry */

typedef struct {
    int64_t x, y;
} pt;

static i128 cross3(pt a, pt b, pt c) {
    /* include/chp/geometry.hpp:29-35 */
    return ((i128)b.x - a.x) * ((i128)c.y - a.y) - ((i128)b.y - a.y) * ((i128)c.x - a.x);
}
static int orient(pt a, pt b, pt c) {
    const i128 v = cross3(a, b, c);
    return v > 0 ? 1 : (v < 0 ? -1 : 0);
}
static i128 dist2(pt a, pt b) {
    const i128 dx = (i128)b.x - a.x, dy = (i128)b.y - a.y;
    return dx * dx + dy * dy;
}
static int lex_less(pt a, pt b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }
static int pt_eq(pt a, pt b) { return a.x == b.x && a.y == b.y; }
static pt get(const int32_t* xy, int64_t i) {
    pt p = {xy[2 * i], xy[2 * i + 1]};
    return p;
}
static void put(int32_t* xy, int64_t i, pt p) {
    xy[2 * i] = (int32_t)p.x;
    xy[2 * i + 1] = (int32_t)p.y;
}

/* degenerate_hull, src/geometry.cpp:29-38 */
static int64_t degenerate(const pt* v, int64_t m, int32_t* out) {
    pt lo = v[0], hi = v[0];
    for (int64_t i = 0; i < m; ++i) {
        if (lex_less(v[i], lo)) lo = v[i];
        if (lex_less(hi, v[i])) hi = v[i];
    }
    put(out, 0, lo);
    if (pt_eq(lo, hi)) return 1;
    put(out, 1, hi);
    return 2;
}

static int64_t canonicalize_pts(pt* v, int64_t m_in, int32_t* out) {
    /* canonicalize_hull, src/geometry.cpp:42-80 */
    int64_t m = 0;
    for (int64_t i = 0; i < m_in; ++i)
        if (m == 0 || !pt_eq(v[m - 1], v[i])) v[m++] = v[i];
    while (m > 1 && pt_eq(v[0], v[m - 1])) --m;
    if (m <= 2) {
        for (int64_t i = 0; i < m; ++i) put(out, i, v[i]);
        return m;
    }
    i128 area = 0;
    for (int64_t i = 0; i < m; ++i) {
        const pt a = v[i], b = v[(i + 1) % m];
        area += (i128)a.x * b.y - (i128)b.x * a.y;
    }
    if (area == 0) return degenerate(v, m, out);
    if (area < 0)
        for (int64_t i = 0, j = m - 1; i < j; ++i, --j) {
            pt t = v[i];
            v[i] = v[j];
            v[j] = t;
        }
    pt* kept = (pt*)malloc((size_t)m * sizeof(pt));
    int changed = 1;
    while (changed && m > 2) {
        changed = 0;
        int64_t k = 0;
        for (int64_t i = 0; i < m; ++i) {
            const pt prev = v[(i + m - 1) % m], next = v[(i + 1) % m];
            if (orient(prev, v[i], next) != 0)
                kept[k++] = v[i];
            else
                changed = 1;
        }
        memcpy(v, kept, (size_t)k * sizeof(pt));
        m = k;
    }
    free(kept);
    if (m <= 2) return degenerate(v, m, out);
    int64_t start = 0;
    for (int64_t i = 1; i < m; ++i)
        if (lex_less(v[i], v[start])) start = i;
    for (int64_t i = 0; i < m; ++i) put(out, i, v[(start + i) % m]);
    return m;
}

int64_t or_canonicalize(const int32_t* v_xy, int64_t m, int32_t* out) {
    if (m <= 0) return -1;
    pt* v = (pt*)malloc((size_t)m * sizeof(pt));
    for (int64_t i = 0; i < m; ++i) v[i] = get(v_xy, i);
    const int64_t h = canonicalize_pts(v, m, out);
    free(v);
    return h;
}

int64_t or_melkman(const int32_t* c, int64_t s, int32_t* out) {
    /* melkman, src/hulls.cpp:137-181 */
    if (s <= 0) return -1;
    pt a = get(c, 0);
    int64_t i = 1;
    while (i < s && pt_eq(get(c, i), a)) ++i;
    if (i == s) {
        put(out, 0, a);
        return 1;
    }
    pt b = get(c, i++);
    while (i < s && orient(a, b, get(c, i)) == 0) {
        const pt vi = get(c, i);
        if (dist2(a, vi) > dist2(a, b))
            b = vi;
        else if (dist2(b, vi) > dist2(a, b))
            a = vi;
        ++i;
    }
    if (i == s) {
        pt two[2] = {a, b};
        return canonicalize_pts(two, 2, out);
    }
    const pt c0 = get(c, i++);
    /* deque as a window [head, tail) into a buffer with room on both ends */
    const int64_t cap = 2 * s + 16;
    pt* buf = (pt*)malloc((size_t)cap * sizeof(pt));
    int64_t head = s + 4, tail = head;
    buf[tail++] = c0;
    if (orient(a, b, c0) > 0) {
        buf[tail++] = a;
        buf[tail++] = b;
    } else {
        buf[tail++] = b;
        buf[tail++] = a;
    }
    buf[tail++] = c0;
    for (; i < s; ++i) {
        const pt q = get(c, i);
        if (orient(buf[tail - 2], buf[tail - 1], q) > 0 &&
            orient(buf[head], buf[head + 1], q) > 0)
            continue;
        while (tail - head >= 2 && orient(buf[tail - 2], buf[tail - 1], q) <= 0) --tail;
        buf[tail++] = q;
        while (tail - head >= 2 && orient(q, buf[head], buf[head + 1]) <= 0) ++head;
        buf[--head] = q;
    }
    --tail; /* front and back duplicate the last hull point */
    const int64_t h = canonicalize_pts(buf + head, tail - head, out);
    free(buf);
    return h;
}

static int cmp_pt(const void* pa, const void* pb) {
    const pt a = *(const pt*)pa, b = *(const pt*)pb;
    if (lex_less(a, b)) return -1;
    if (lex_less(b, a)) return 1;
    return 0;
}

int64_t or_monotone_hull(const int32_t* xy, int64_t n, int32_t* out) {
    if (n <= 0) return -1;
    pt* p = (pt*)malloc((size_t)n * sizeof(pt));
    for (int64_t i = 0; i < n; ++i) p[i] = get(xy, i);
    qsort(p, (size_t)n, sizeof(pt), cmp_pt);
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
        if (m == 0 || !pt_eq(p[m - 1], p[i])) p[m++] = p[i];
    if (m == 1) {
        put(out, 0, p[0]);
        free(p);
        return 1;
    }
    pt* h = (pt*)malloc((size_t)(2 * m + 2) * sizeof(pt));
    int64_t k = 0;
    for (int64_t i = 0; i < m; ++i) {
        while (k >= 2 && orient(h[k - 2], h[k - 1], p[i]) <= 0) --k;
        h[k++] = p[i];
    }
    const int64_t lower = k + 1;
    for (int64_t i = m - 2; i >= 0; --i) {
        while (k >= lower && orient(h[k - 2], h[k - 1], p[i]) <= 0) --k;
        h[k++] = p[i];
    }
    --k; /* last point repeats the first */
    if (k < 2) k = 2;  /* all collinear: lexmin, lexmax */
    for (int64_t i = 0; i < k; ++i) put(out, i, h[i]);
    free(h);
    free(p);
    return k;
}

void or_min_max(const int32_t* xy, uint64_t n, int64_t out[4]) {
    int64_t xmin = xy[0], xmax = xy[0], ymin = xy[1], ymax = xy[1];
    for (uint64_t i = 1; i < n; ++i) {
        const int64_t x = xy[2 * i], y = xy[2 * i + 1];
        if (x < xmin) xmin = x;
        if (x > xmax) xmax = x;
        if (y < ymin) ymin = y;
        if (y > ymax) ymax = y;
    }
    out[0] = xmin;
    out[1] = xmax;
    out[2] = ymin;
    out[3] = ymax;
}
