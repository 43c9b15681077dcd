/*
 * cdc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU definitions of the hashless CDC
 * operations of PAPER.md (arxiv 2508.05797, "Accelerating Data Chunking in
 * Deduplication Systems using Vector Instructions").  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, table or constant with
 * the CUDA path under paper_2508_05797_b200/ and never calls it.
 *
 * Conventions (DESIGN.md §3 "Readings"):
 *   - a stream is d[0..L); chunks tile it; a chunk starting at s ends at the
 *     exclusive offset e returned by *_chunk_end (the next chunk starts at e);
 *   - max_size caps a chunk's length (reading R5); the paper's hashless
 *     algorithms have no other minimum than the one their window implies
 *     (every content boundary lies >= w bytes after the chunk start);
 *   - window w >= 1 and max_size > w are required (checked by the caller).
 *
 * Every function follows the paper's description step by step; no blocking,
 * fusion or reordering.  Parity is pinned in tests/test_oracle_*.py.
 */
#include <stdint.h>
#include <stddef.h>

enum { OR_MAX = 0, OR_MIN = 1 };
enum { OR_GT = 0, OR_GEQ = 1, OR_LT = 2, OR_LEQ = 3, OR_EQ = 4 };
enum { OR_RAM = 0, OR_AE_MAX = 1, OR_AE_MIN = 2, OR_MAXP = 3 };

/*
 * Extreme Byte Search -- PAPER.md §4.1 (lines 324-330): "identifies the
 * extreme byte (maximum/minimum) in a fixed-size window".  The paper returns
 * only the value; we also return the leftmost position holding it (reading R6).
 * Returns 0 on success, -1 for an empty region.
 */
int oracle_extreme_byte_search(const uint8_t *region, uint64_t n, int mode,
                               uint8_t *value, uint64_t *pos)
{
    if (n == 0)
        return -1;
    uint8_t best = region[0];
    uint64_t best_pos = 0;
    for (uint64_t i = 1; i < n; i++) {
        int better = (mode == OR_MAX) ? (region[i] > best) : (region[i] < best);
        if (better) {
            best = region[i];
            best_pos = i;
        }
    }
    *value = best;
    *pos = best_pos;
    return 0;
}

static int cmp_holds(uint8_t b, uint8_t target, int cmp)
{
    switch (cmp) {
    case OR_GT:  return b > target;
    case OR_GEQ: return b >= target;
    case OR_LT:  return b < target;
    case OR_LEQ: return b <= target;
    default:     return b == target;
    }
}

/*
 * Range Scan -- PAPER.md §4.2 (lines 343-347): "bytes are serially compared
 * against a target value" with one of the comparators GT, GEQ, LT, LEQ, EQ.
 * Returns the index of the first byte b with (b cmp target), or n if none.
 */
uint64_t oracle_range_scan(const uint8_t *region, uint64_t n, uint8_t target, int cmp)
{
    for (uint64_t i = 0; i < n; i++)
        if (cmp_holds(region[i], target, cmp))
            return i;
    return n;
}

/*
 * RAM -- PAPER.md §2.1.2 (line 198, Fig. 2c) and §4.3 (line 355):
 * "RAM begins by scanning a fixed-size window at the beginning of each chunk
 * to find the maximum valued byte (F1).  It then begins scanning at the first
 * byte outside the window, serially comparing these bytes against this
 * maximum value.  A chunk boundary is inserted when the first byte that
 * exceeds or equals the maximum is found (F3)."  The boundary byte is the
 * last byte of the chunk (reading R2).
 */
uint64_t oracle_ram_chunk_end(const uint8_t *d, uint64_t L, uint64_t s,
                              uint64_t w, uint64_t max_size)
{
    if (L - s <= w)                       /* window does not fit: final chunk */
        return L;
    uint8_t M;
    uint64_t mpos;
    oracle_extreme_byte_search(d + s, w, OR_MAX, &M, &mpos);   /* window [s, s+w) */
    uint64_t limit = (L - s < max_size) ? L : s + max_size;     /* R5 cap */
    uint64_t i = s + w + oracle_range_scan(d + s + w, limit - (s + w), M, OR_GEQ);
    if (i < limit)
        return i + 1;                     /* boundary byte d[i] ends the chunk */
    return limit;                         /* max_size cap, or end of stream */
}

/*
 * AE-Max / AE-Min -- PAPER.md §2.1.2 (lines 169-171, Fig. 2a) and §4.3
 * (lines 357-359): find a target byte greater (AE-Max) / less (AE-Min) than
 * all the bytes before it in the chunk; scan the fixed-size window of w bytes
 * after the target for its maximum (minimum); if the target is not exceeded
 * by that extreme (reading R1) insert a boundary after the window, otherwise
 * "scanning continues for a new target byte" with a GT (LT) Range Scan.
 *
 * The first byte of a chunk has no byte before it and so is the first target.
 * Because the current target t holds the running extreme of d[s..t], the next
 * target is the first byte after t that strictly exceeds d[t]; when the window
 * test fails that byte lies inside the window (its extreme exceeds d[t]).
 */
uint64_t oracle_ae_chunk_end(const uint8_t *d, uint64_t L, uint64_t s,
                             uint64_t w, uint64_t max_size, int mode)
{
    uint64_t limit = (L - s < max_size) ? L : s + max_size;     /* R5 cap */
    uint64_t t = s;                                             /* first target */
    for (;;) {
        /* the boundary would be the window's last byte d[t+w]; it must lie
         * inside the chunk limit, and no later target can end earlier */
        if (t + w >= limit)
            return limit;
        uint8_t ext;
        uint64_t epos;
        oracle_extreme_byte_search(d + t + 1, w, mode, &ext, &epos);  /* window (t, t+w] */
        int target_wins = (mode == OR_MAX) ? (d[t] >= ext) : (d[t] <= ext);
        if (target_wins)
            return t + w + 1;                 /* boundary after the window */
        int cmp = (mode == OR_MAX) ? OR_GT : OR_LT;
        t = t + 1 + oracle_range_scan(d + t + 1, w, d[t], cmp);   /* next target */
    }
}

/*
 * MAXP -- PAPER.md §2.1.2 (line 173, Fig. 2b, and line 196) and §4.3 (line
 * 361): "MAXP identifies target bytes in the data stream that are local
 * maxima, i.e., they are greater than a fixed number of bytes before and
 * after them.  When such target bytes are found, chunk boundaries are
 * inserted at their locations"; "MAXP works by sliding two fixed-size windows
 * over the data, tracking the maximum values from both windows.  These
 * windows are located one byte apart ... and the byte between them is the
 * target byte.  When the target byte's value is greater than the maximum
 * value from both windows, a chunk boundary is inserted"; "A chunk boundary
 * is inserted right after such a byte is found".
 *
 * Readings (M1-M4): the two windows hold h = w bytes each,
 * [t-h, t) and (t, t+h], and the test is strict (M1); the target is the last
 * byte of its chunk (M2, as R2); the left window starts at the chunk start,
 * so the first target examined is s + h (M3); the right window must lie
 * inside the stream (M4); max_size caps the chunk (R5).
 *
 * "greater than the maximum value from both windows" is "greater than every
 * byte of both windows"; the loop below stops at the first window byte that
 * is not smaller, which decides the same predicate.
 */
static int oracle_maxp_is_target(const uint8_t *d, uint64_t L, uint64_t t, uint64_t h)
{
    if (t < h || t + h >= L)              /* both windows must lie in the stream */
        return 0;
    for (uint64_t j = 1; j <= h; j++)
        if (d[t - j] >= d[t] || d[t + j] >= d[t])
            return 0;
    return 1;
}

uint64_t oracle_maxp_chunk_end(const uint8_t *d, uint64_t L, uint64_t s,
                               uint64_t h, uint64_t max_size)
{
    uint64_t limit = (L - s < max_size) ? L : s + max_size;     /* R5 cap */
    for (uint64_t t = s + h; t < limit; t++)                     /* chunk [s, t+1) fits */
        if (oracle_maxp_is_target(d, L, t, h))
            return t + 1;                                        /* boundary right after the target */
    return limit;
}

uint64_t oracle_chunk_end(int algo, const uint8_t *d, uint64_t L, uint64_t s,
                          uint64_t w, uint64_t max_size)
{
    if (algo == OR_MAXP)
        return oracle_maxp_chunk_end(d, L, s, w, max_size);
    if (algo == OR_RAM)
        return oracle_ram_chunk_end(d, L, s, w, max_size);
    return oracle_ae_chunk_end(d, L, s, w, max_size,
                               algo == OR_AE_MAX ? OR_MAX : OR_MIN);
}

/*
 * Whole-stream chunking: the chain s_0 = 0, s_{j+1} = chunk_end(s_j) until L.
 * Writes the exclusive chunk end offsets (the last one is L) into out[] and
 * returns their number (0 for an empty stream); stops early at cap entries.
 */
uint64_t oracle_chunk(int algo, const uint8_t *d, uint64_t L, uint64_t w,
                      uint64_t max_size, uint64_t *out, uint64_t cap)
{
    uint64_t n = 0, s = 0;
    while (s < L && n < cap) {
        uint64_t e = oracle_chunk_end(algo, d, L, s, w, max_size);
        out[n++] = e;
        s = e;
    }
    return n;
}

/*
 * The chain from an arbitrary start (used by tests of the speculative /
 * range-sharded host logic): starts at `start` as if a chunk began there and
 * records every chunk start in [start, stop) followed by the first start >= stop
 * (or L).  Returns the number written.
 */
uint64_t oracle_chain_from(int algo, const uint8_t *d, uint64_t L, uint64_t start,
                           uint64_t stop, uint64_t w, uint64_t max_size,
                           uint64_t *out, uint64_t cap)
{
    uint64_t n = 0, s = start;
    while (n < cap) {
        out[n++] = s;
        if (s >= stop || s >= L)
            break;
        s = oracle_chunk_end(algo, d, L, s, w, max_size);
    }
    return n;
}

/*
 * Verification of a chunking produced elsewhere (the CUDA path) against the
 * definition above, one chunk at a time so that callers can split the work
 * over host threads.  ends[0..n) is a chunking of d[0..L) exactly when
 * ends[0] = chunk_end(0), ends[j] = chunk_end(ends[j-1]) for every j, and
 * ends[n-1] = L -- i.e. when it equals what oracle_chunk writes (the chain is
 * determined by its start, §2.1.2: each boundary depends only on the bytes
 * after the chunk start).  This checks entries [j0, j1): returns the first j
 * in that range with ends[j] != chunk_end(j ? ends[j-1] : 0), or j1.
 */
uint64_t oracle_check_ends(int algo, const uint8_t *d, uint64_t L, uint64_t w,
                           uint64_t max_size, const uint64_t *ends,
                           uint64_t j0, uint64_t j1)
{
    for (uint64_t j = j0; j < j1; j++) {
        uint64_t s = j ? ends[j - 1] : 0;
        if (s >= L || oracle_chunk_end(algo, d, L, s, w, max_size) != ends[j])
            return j;
    }
    return j1;
}

/*
 * The same for files [f0, f1) of a packed batch: file f is
 * d[offs[f] .. offs[f+1]) and its ends (relative to the file start) are
 * ends[bo[f] .. bo[f+1]).  A file is correct when its ends pass
 * oracle_check_ends and the last one equals its length (none for an empty
 * file).  Returns the first wrong file, or f1; *bad_j receives the index of
 * the first wrong entry within that file's ends (its count if the entries
 * are right but the count is not).
 */
uint64_t oracle_check_batch(int algo, const uint8_t *d, const uint64_t *offs,
                            const uint64_t *ends, const uint64_t *bo,
                            uint64_t f0, uint64_t f1, uint64_t w,
                            uint64_t max_size, uint64_t *bad_j)
{
    for (uint64_t f = f0; f < f1; f++) {
        uint64_t L = offs[f + 1] - offs[f];
        uint64_t n = bo[f + 1] - bo[f];
        const uint64_t *e = ends + bo[f];
        uint64_t j = oracle_check_ends(algo, d + offs[f], L, w, max_size, e, 0, n);
        if (j < n) {
            *bad_j = j;
            return f;
        }
        if ((L == 0) != (n == 0) || (n > 0 && e[n - 1] != L)) {
            *bad_j = n;
            return f;
        }
    }
    return f1;
}
