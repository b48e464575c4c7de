/*
 * chp_oracle.h -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_1505_00914_b200/ links, loads
 * or calls this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and only as the checker.
 *
 * Every function restates one piece of the reference (paths relative to
 * /root/reference/proj) in plain C11 with exact integer arithmetic
 * (__int128 cross products, as include/chp/geometry.hpp:29-35 does).
 *
 * Parity pin: the restatement is checked against
 *   (1) the reference's own KATs (tests/test_reducer.cpp, tests/test_hulls.cpp),
 *   (2) the config-1 golden digests of SURVEY.md Appendix A, produced by the
 *       reference itself, and
 *   (3) oracle/_ref/libchpref.so -- the reference's sources compiled here by
 *       oracle/Makefile -- on randomized inputs (tests/test_oracle.py).
 */
#ifndef CHP_ORACLE_H
#define CHP_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FNV-1a-64 over raw bytes (SURVEY.md Appendix A digest definition). */
uint64_t or_fnv1a64(const void* data, size_t len);

/* std::mt19937_64 + libstdc++ uniform_int_distribution<int64_t>(1,p):
 * the reference "uniform-box" generator, src/dataset.cpp:35-59 (x drawn
 * before y, :59).  Writes n interleaved int32 (x,y) pairs. */
void or_gen_uniform_box(uint64_t n, int64_t p, uint64_t seed, int32_t* xy);

/* reducer::reduce, src/reducer.cpp:69-79: validation pass (:72-75) then
 * the Algorithm-1 fold `bucket` (:19-32).  lo/hi/valid have `width`
 * entries, occ has ceil(width/64) words in BlockedBitset<uint64_t> layout
 * (include/chp/occupancy.hpp:46-49, :70-74).  q < 0 means "no q".
 * Returns 0, or -1 when the reference would throw std::invalid_argument. */
int or_reduce(const int32_t* xy, uint64_t n, int64_t width, int64_t q,
              int32_t* lo, int32_t* hi, uint8_t* valid, uint64_t* occ);

/* The fold alone on pre-translated points (no validation), accumulating
 * into existing arrays: bucket() with slot = x - x_off - 1
 * (src/reducer.cpp:19-32, translation as in :160-168). */
void or_bucket(const int32_t* xy, uint64_t n, int64_t x_off, int32_t* lo,
               int32_t* hi, uint8_t* valid, uint64_t* occ);

/* SURVEY.md 8(c) chunked procedure: reduce() per slice on host threads,
 * merged slot by slot into the caller's (lo, hi, valid) accumulator
 * (initialise valid to 0 once).  Returns 0 or -1 (invalid coordinate). */
int or_reduce_accumulate_mt(const int32_t* xy, uint64_t n, int64_t width, int64_t q,
                            int threads, int32_t* lo, int32_t* hi, uint8_t* valid);

/* Occupancy words of a merged array (Index::insert per valid slot). */
void or_occ_from_valid(int64_t width, const uint8_t* valid, uint64_t* occ);

/* L in int32 (lo,hi) pairs, empty slots as the (width+1,-1) sentinel of
 * serialize(), src/reducer.cpp:121-130. */
void or_L_pairs(int64_t width, const int32_t* lo, const int32_t* hi,
                const uint8_t* valid, int32_t* out_pairs);

/* serialize() text, src/reducer.cpp:121-130.  Returns bytes written (or
 * needed, when buf is NULL). */
size_t or_serialize(int64_t width, const int32_t* lo, const int32_t* hi,
                    const uint8_t* valid, char* buf, size_t cap);

/* ExtremalArray::valid_count, src/reducer.cpp:42-49. */
int64_t or_valid_count(int64_t width, const int32_t* lo, const int32_t* hi,
                       const uint64_t* occ);

/* build_polyline, src/reducer.cpp:108-119: ctz walk of the occupancy words
 * (include/chp/occupancy.hpp:83-93) emitting to_original(i,lo) then
 * to_original(i,hi) when hi != lo (include/chp/reducer.hpp:46-50).
 * Returns the chain length s, or -1 when empty (reference throws). */
int64_t or_build_polyline(int64_t width, const int32_t* lo, const int32_t* hi,
                          const uint64_t* occ, int64_t major_off,
                          int64_t minor_off, int swapped, int32_t* chain_xy);

/* The north_star order (minima by increasing x, then maxima by decreasing
 * x, the max only when hi != lo).  No reference function produces it;
 * restated per SURVEY.md 8(c) from the same ExtremalArray. */
int64_t or_ns_chain(int64_t width, const int32_t* lo, const int32_t* hi,
                    const uint64_t* occ, int64_t major_off, int32_t* chain_xy);

/* hulls::melkman, src/hulls.cpp:137-181, finished by canonicalize_hull,
 * src/geometry.cpp:42-80.  Returns h, or -1 on empty input. */
int64_t or_melkman(const int32_t* chain_xy, int64_t s, int32_t* hull_xy);

/* canonicalize_hull, src/geometry.cpp:42-80 (in/out may not alias). */
int64_t or_canonicalize(const int32_t* v_xy, int64_t m, int32_t* hull_xy);

/* Andrew monotone chain on the lex-sorted unique points, strict, CCW from
 * the lex-min vertex -- an independent cross-check of or_melkman (equal to
 * graham_scan, src/hulls.cpp:34-61, on every input). */
int64_t or_monotone_hull(const int32_t* xy, int64_t n, int32_t* hull_xy);

/* kernels::min_max_scalar, src/kernels.cpp:8-17. n >= 1. */
void or_min_max(const int32_t* xy, uint64_t n, int64_t out4[4]);

#ifdef __cplusplus
}
#endif
#endif
