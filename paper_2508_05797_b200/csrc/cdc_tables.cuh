// cdc_tables.cuh -- transfer tables for saturated streams (T-mode).
// Included once by cdc_kernels.cu inside namespace cdc, after the workspace
// (Work), the segment geometry (SegInfo) and the look-back words it uses.
#pragma once

// ------------------------------------------------------------------ T-mode: transfer tables
// (DESIGN.md §6).  On saturating data (uniform bytes at w >> 256) chains that
// start at different offsets meet only after ~(w / 362)^2 chunks, so halo
// walks get long.  There a chunk step depends only on the positions of the
// saturating bytes (255 for RAM and AE-Max, 0 for AE-Min):
//   RAM (§2.1.2): the window [x, x+w) holds a saturating byte, so its maximum
//     is saturated and the chunk ends after the first saturating byte in
//     [x+w, limit), else at limit;
//   AE: the first saturating byte q <= x+w is the target no byte beats (every
//     earlier record is beaten within w), so the chunk ends at q+w+1, or at
//     limit when q+w >= limit; if x+w >= limit it ends at limit.
// A saturated chain that enters segment g starts at one of few candidates
// (RAM: P+1 for a saturating position P in [p_g - 1, N(p_g + w - 1)]; AE:
// q+w+1 for q in [p_g - w - 1, N(p_g - 1)], N = next saturating position;
// segment 0: the stream start).  Before any byte walk, walker g looks at its
// first 16 KiB; if they are dense in saturating bytes it indexes those of
// [p_g - w - 1, t_ihi) (and the long constant runs) in its
// idle ring, walks every candidate's chain in index space (one lane each;
// the few steps the index cannot decide are read from the bytes) and
// publishes, per candidate, the number of chain starts inside the segment and
// the candidate of segment g+1 its chain enters -- or, when its exit is no
// candidate, hands that exit over as an extra entry of segment g+1.  The last
// walker of each block of 32 segments composes the block's tables with
// shuffles, the last composer scans the blocks, and every walker writes its
// own part of the true chain: no byte walk and no halo.  Anything the tables
// cannot resolve makes the whole call fall back to the speculative walk (the
// tables are tried only for a single stream whose grid is one co-resident
// wave, with a timeout).  DESIGN.md §6 lists every case.
constexpr int TK = 128;                      // table rows per segment (candidates + extra entries), 4 per lane
constexpr int TEX = 64;                      // extra entries a segment can pass to the next one
constexpr int TRUNS = 16;                    // constant runs a walker records (tail of its ring)
constexpr uint32_t T_RUN_WORDS = 2 + 3 * TRUNS;  // count, TRUNS x (start, end, value), longest run
#ifndef CDC_T_LONG_RUN
#define CDC_T_LONG_RUN 32768
#endif
constexpr uint32_t T_LONG_RUN = CDC_T_LONG_RUN;  // a constant run this long makes the attempt give up at once
constexpr uint32_t T_END = 0xFFFFFFFEu;      // link: the chain reached the stream end
constexpr uint32_t T_BAD = 0xFFFFFFFFu;      // link: not resolvable in index space
constexpr uint32_t T_DENSE = 8;              // saturating bytes per window a segment needs
constexpr uint32_t T_IDX_CAP = (uint32_t)(RING_BYTES / 4);
constexpr uint32_t T_IX_CAP = T_IDX_CAP - T_RUN_WORDS;  // index entries; the constant runs follow them
constexpr unsigned long long T_TIMEOUT_NS = 2000000ull;  // the scanner gives up after 2 ms
// one segment per CTA (t_coop_index): the idle rings of warps 1.. keep every
// row's chain starts (offsets from p, entry j of row k at [j * TK + k]), so
// the write after the verdict is a copy instead of a second walk
constexpr int TPOS = 64;
static_assert((SPEC_WARPS - 1) * RING_SMEM >= TK * TPOS * 4, "chain-start store does not fit the idle rings");
// control words (ctrl[], reset to ~0 by k_reset): 6 block composers arrived,
// 7 all-T (~0 yes, 0 no), 8 verdict (~0 pending, 1 tables, 0 fall back)
constexpr int T_ARRIVE = 6, T_ALL = 7, T_SCAN = 8;

// ctrl[12], ctrl[13]: the first failure's reason and segment (diagnostics,
// printed by cdc_stats when CDC_TDEBUG is set)
__device__ __forceinline__ void t_fail(Work &W, uint32_t why = 0, uint64_t g = 0) {
    if (ld_relaxed_u32(W.ctrl + T_ALL) != 0u) atomicAnd(W.ctrl + T_ALL, 0u);
    if (why && atomicCAS(W.ctrl + 12, ~0u, why) == ~0u) W.ctrl[13] = (uint32_t)g;
}
__device__ __forceinline__ bool t_alive(const Work &W) { return ld_relaxed_u32(W.ctrl + T_ALL) != 0u; }

// index of the saturating bytes of the file positions [lo, hi): ascending
// offsets from rel into ix; returns the count, cap + 1 when they do not fit (or the attempt is off), cap + 2 at a constant run of T_LONG_RUN bytes.
// Each lane takes TIX_G contiguous granules of 16 bytes, so lane order is
// position order and one warp scan of the lanes' counts places every entry.
// any byte of a 16-byte vector equal to the saturating value (255 for MAX, 0
// for MIN): the zero-byte test on ~x (MAX) or x (MIN), exact for "any"
template <bool MAX>
__device__ __forceinline__ bool t_sat_any(const uint4 &v) {
    auto f = [](uint32_t x) {
        return MAX ? (0xFEFEFEFEu - x) & x & 0x80808080u : (x - 0x01010101u) & ~x & 0x80808080u;
    };
    return (f(v.x) | f(v.y) | f(v.z) | f(v.w)) != 0u;
}
#ifndef CDC_TIX_G
#define CDC_TIX_G 16
#endif
constexpr int TIX_G = CDC_TIX_G;  // 16-byte granules per lane per step of the index pass
#ifndef CDC_TIX_PF
#define CDC_TIX_PF 2
#endif
constexpr int TIX_PF = CDC_TIX_PF;  // steps ahead the index pass asks the TMA unit to bring into L2
// bulk L2 prefetch of [p, min(p + bytes, end)) (one lane; p 16-byte aligned)
__device__ __forceinline__ void t_prefetch_l2(uintptr_t p, uintptr_t end, uint32_t bytes) {
    if (p >= end) return;
    const uint32_t sz = (uint32_t)(end - p < bytes ? end - p : bytes) & ~15u;
    if (sz) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(sz) : "memory");
}
template <bool MAX>
__device__ uint32_t t_index(const uint8_t *fbase, int64_t lo, int64_t hi, int64_t rel, uint32_t *ix, uint32_t cap,
                            const uint32_t *alive = nullptr, uint32_t *runs = nullptr) {
    const int lane = lane_id();
    const uintptr_t fb = reinterpret_cast<uintptr_t>(fbase);
    const uintptr_t a0 = (fb + (uintptr_t)lo) & ~(uintptr_t)15;
    const uintptr_t a1 = fb + (uintptr_t)hi;
    uint32_t n = 0;
    int step = 0;
    // constant runs (whole 8 KiB steps of one repeated byte): lane 0 tracks the open one
    uint32_t nr = 0, rs = 0, re = 0, rc = 0, longest = 0;
    bool ropen = false;
    auto close_run = [&]() {
        if (ropen && re - rs > longest) longest = re - rs;
        if (ropen && nr < (uint32_t)TRUNS && lane == 0) {
            runs[1 + 3 * nr] = rs;
            runs[2 + 3 * nr] = re;
            runs[3 + 3 * nr] = rc;
        }
        if (ropen && nr < (uint32_t)TRUNS) ++nr;
        ropen = false;
    };
    constexpr uint32_t BLK = 32 * 16 * TIX_G;
    if (TIX_PF > 0 && lane == 0)
        for (int k = 1; k < TIX_PF; ++k) t_prefetch_l2(a0 + (uintptr_t)k * BLK, a1, BLK);
    for (uintptr_t a = a0; a < a1; a += BLK) {
        if (TIX_PF > 0 && lane == 0) t_prefetch_l2(a + (uintptr_t)TIX_PF * BLK, a1, BLK);
        // the attempt may already have failed elsewhere: look every 16 KiB
        if (alive && (++step & 1) == 0 && ld_relaxed_u32(alive) == 0u) return cap + 1;
        const uintptr_t la = a + (uintptr_t)lane * 16 * TIX_G;
        // pass 1: which granules hold a saturating byte (2 integer ops per word;
        // a flag may sit in a byte outside [lo, hi), the exact pass drops it)
        uint32_t hit = 0;
        uint32_t crep = 0;
        bool lconst = runs != nullptr;
#pragma unroll
        for (int u = 0; u < TIX_G; ++u) {
            const uintptr_t ga = la + (uintptr_t)(u * 16);
            if (ga < a1) {
                const uint4 v = *reinterpret_cast<const uint4 *>(ga);
                if (u == 0) crep = (v.x & 0xFFu) * 0x01010101u;
                lconst = lconst && ((v.x ^ crep) | (v.y ^ crep) | (v.z ^ crep) | (v.w ^ crep)) == 0u;
                if (t_sat_any<MAX>(v)) hit |= 1u << u;
            } else {
                lconst = false;
            }
        }
        // exact byte mask of hit granule u inside [lo, hi) (reloaded: an L1 hit)
        auto exact = [&](int u) -> uint32_t {
            const uintptr_t ga = la + (uintptr_t)(u * 16);
            const uint4 v = *reinterpret_cast<const uint4 *>(ga);
            const int64_t pos = (int64_t)(ga - fb);
            const int x0 = (int)(lo - pos > 0 ? (lo - pos > 16 ? 16 : lo - pos) : 0);
            const int x1 = (int)(hi - pos < 16 ? (hi - pos < 0 ? 0 : hi - pos) : 16);
            const uint32_t keep = x0 < x1 ? (((1u << x1) - 1u) & ~((1u << x0) - 1u)) : 0u;
            return sat_mask16<MAX>(v) & keep;
        };
        if (runs != nullptr) {
            const int64_t s0 = (int64_t)(a - fb), s1 = s0 + 32 * 16 * TIX_G;
            const uint32_t c0rep = __shfl_sync(0xFFFFFFFFu, crep, 0);  // every lane, before any branch
            const bool whole = __all_sync(0xFFFFFFFFu, lconst && crep == c0rep) && s0 >= lo && s1 <= hi;
            const uint32_t c8 = c0rep & 0xFFu;
            if (whole) {
                if (ropen && rc == c8 && (int64_t)re + rel == s0) {
                    re = (uint32_t)(s1 - rel);
                    if (re - rs >= T_LONG_RUN) return cap + 2;  // a long constant run: give up at once
                } else {
                    close_run();
                    ropen = true;
                    rs = (uint32_t)(s0 - rel);
                    re = (uint32_t)(s1 - rel);
                    rc = c8;
                }
            } else {
                close_run();
            }
        }
        uint32_t c = 0;
        for (uint32_t h = hit; h; h &= h - 1u) c += __popc(exact(__ffs(h) - 1));
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if (n + tot > cap) return cap + 1;
        uint32_t at = n + incl - c;
        const uint32_t base = (uint32_t)((int64_t)(la - fb) - rel);
        for (uint32_t h = hit; h; h &= h - 1u) {
            const int u = __ffs(h) - 1;
            uint32_t mm = exact(u);
            while (mm) {
                ix[at++] = base + (uint32_t)(u * 16) + (uint32_t)(__ffs(mm) - 1);
                mm &= mm - 1u;
            }
        }
        n += tot;
    }
    if (runs != nullptr) {
        close_run();
        if (lane == 0) {
            runs[0] = nr;
            runs[1 + 3 * TRUNS] = longest;
        }
    }
    __syncwarp();
    return n;
}

#ifdef CDC_T_CONST_SAMPLE
// (experiment) true when the bytes [a, b) all equal: a density sample inside a
// zero-filled region is then accepted.  Warp-cooperative.
__device__ bool t_constant(const uint8_t *fbase, int64_t a, int64_t b) {
    const uintptr_t fb = reinterpret_cast<uintptr_t>(fbase);
    const uint32_t c = fbase[a] * 0x01010101u;
    bool same = true;
    for (uintptr_t ga = ((fb + (uintptr_t)a) & ~(uintptr_t)15) + (uintptr_t)lane_id() * 16; ga < fb + (uintptr_t)b;
         ga += 32 * 16) {
        const uint4 v = *reinterpret_cast<const uint4 *>(ga);
        const int64_t pos0 = (int64_t)(ga - fb);
        if (pos0 >= a && pos0 + 16 <= b) same = same && ((v.x ^ c) | (v.y ^ c) | (v.z ^ c) | (v.w ^ c)) == 0u;
    }
    return __all_sync(0xFFFFFFFFu, same);
}
#endif

// Bucket table over the index (in the ring's free words below the constant
// runs): bk[c] = the first entry >= c * 256, so a lookup reads two bucket
// words and about one entry instead of a dozen dependent loads of a binary
// search.  ix[T_IX_CAP - 1] holds the bucket count (0: no table) whenever
// n < T_IX_CAP; the u16 buckets sit just below it.
constexpr int T_BK_SHIFT = 8;
__device__ __forceinline__ const uint16_t *t_bk(const uint32_t *ix, uint32_t nb) {
    return reinterpret_cast<const uint16_t *>(ix + T_IX_CAP - 1 - (nb + 1) / 2);
}
// (all lanes; after the index is final) span = ihi - lo
__device__ void t_buckets(uint32_t *ix, uint32_t n, int64_t span) {
    if (n >= T_IX_CAP) return;  // the header word is an entry (and such an index is refused anyway)
    const int lane = lane_id();
    const uint32_t nb = (uint32_t)(span >> T_BK_SHIFT) + 1;
    const bool fit = (uint64_t)n + 1 + (nb + 1) / 2 <= (uint64_t)T_IX_CAP;
    if (fit) {
        uint16_t *bk = const_cast<uint16_t *>(t_bk(ix, nb));
        for (uint32_t i = lane; i < n; i += 32) {
            const uint32_t c0 = i == 0 ? 0u : (ix[i - 1] >> T_BK_SHIFT) + 1;
            const uint32_t c1 = ix[i] >> T_BK_SHIFT;
            for (uint32_t c = c0; c <= c1; ++c) bk[c] = (uint16_t)i;
        }
        const uint32_t t0 = n == 0 ? 0u : (ix[n - 1] >> T_BK_SHIFT) + 1;
        for (uint32_t c = t0 + lane; c < nb; c += 32) bk[c] = (uint16_t)n;
    }
    __syncwarp();
    if (lane == 0) ix[T_IX_CAP - 1] = fit ? nb : 0u;
    __syncwarp();
}

// first entry of ix[0..n) that is >= r
__device__ __forceinline__ uint32_t t_lb(const uint32_t *ix, uint32_t n, uint32_t r) {
    uint32_t a = 0, b = n;
    const uint32_t nb = n < T_IX_CAP ? ix[T_IX_CAP - 1] : 0u;
    if (nb != 0u) {
        const uint32_t c = r >> T_BK_SHIFT;
        if (c >= nb) return n;
        const uint16_t *bk = t_bk(ix, nb);
        a = bk[c];
        const uint32_t e = c + 1 < nb ? bk[c + 1] : n;
        while (a < e && ix[a] < r) ++a;
        return a;
    }
    while (a < b) {
        const uint32_t m = (a + b) >> 1;
        if (ix[m] < r) a = m + 1;
        else b = m;
    }
    return a;
}

// one saturated chunk step from start x (one lane); -1 when the step is not
// saturated or needs bytes outside the index [lo, ihi)
template <int ALGO>
__device__ __forceinline__ int64_t t_step(const uint32_t *ix, uint32_t n, int64_t lo, int64_t ihi, int64_t x,
                                          int64_t w, int64_t mx, int64_t Lf) {
    const int64_t limit = Lf - x < mx ? Lf : x + mx;
    if constexpr (ALGO == ALGO_RAM) {
        if (x + w >= Lf) return Lf;  // the window does not fit: a single final chunk
        if (x + w > ihi) return -1;
        const uint32_t i1 = t_lb(ix, n, (uint32_t)(x - lo));
        if (i1 >= n || lo + (int64_t)ix[i1] >= x + w) return -1;  // the window holds no saturating byte
        const uint32_t i2 = t_lb(ix, n, (uint32_t)(x + w - lo));
        if (i2 < n && lo + (int64_t)ix[i2] < limit) return lo + (int64_t)ix[i2] + 1;
        return limit <= ihi ? limit : -1;
    } else {
        if (x + w >= limit) return limit;
        if (x + w + 1 > ihi) return -1;
        const uint32_t i = t_lb(ix, n, (uint32_t)(x - lo));
        if (i >= n) return -1;
        const int64_t q = lo + (int64_t)ix[i];
        if (q > x + w) return -1;  // no saturating byte within w: not a saturated step
        return q + w < limit ? q + w + 1 : limit;
    }
}

// One chunk step from start x read from the bytes themselves (one lane, any
// data): the rules of PAPER.md §2.1.2 exactly as run_chain applies them, for
// the steps the index cannot decide (a window without a saturating byte, e.g.
// inside a zero-filled region).  16-byte loads, a byte-extreme test per
// granule, a byte loop only in the granule that holds the answer.
template <bool MAX>
__device__ __forceinline__ uint4 t_granule(const uint8_t *fbase, uintptr_t ga, int64_t a, int64_t b, int64_t &pos0) {
    uint4 v = *reinterpret_cast<const uint4 *>(ga);
    pos0 = (int64_t)(ga - reinterpret_cast<uintptr_t>(fbase));
    if (pos0 < a || pos0 + 16 > b) {  // neutralise the bytes outside [a, b)
        const int x0 = (int)(a - pos0 > 0 ? (a - pos0 > 16 ? 16 : a - pos0) : 0);
        const int x1 = (int)(b - pos0 < 16 ? (b - pos0 < 0 ? 0 : b - pos0) : 16);
        const uint32_t m16 = x0 < x1 ? (((1u << x1) - 1u) & ~((1u << x0) - 1u)) : 0u;
        uint32_t k[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) k[j] = (((((m16 >> (4 * j)) & 0xFu) * 0x00204081u) & 0x01010101u) * 0xFFu);
        if (MAX) { v.x &= k[0]; v.y &= k[1]; v.z &= k[2]; v.w &= k[3]; }
        else { v.x |= ~k[0]; v.y |= ~k[1]; v.z |= ~k[2]; v.w |= ~k[3]; }
    }
    return v;
}
// extreme of the bytes [a, b) (a < b)
template <bool MAX>
__device__ uint32_t t_bytes_ext(const uint8_t *fbase, int64_t a, int64_t b) {
    const uintptr_t fb = reinterpret_cast<uintptr_t>(fbase);
    uint32_t acc = neutral<MAX>();
    for (uintptr_t ga = (fb + (uintptr_t)a) & ~(uintptr_t)15; ga < fb + (uintptr_t)b; ga += 16) {
        int64_t pos0;
        acc = ext2<MAX>(acc, vext16<MAX>(t_granule<MAX>(fbase, ga, a, b, pos0)));
        if (acc == (MAX ? 255u : 0u)) break;
    }
    return acc;
}
// first position in [a, b) whose byte satisfies (byte CMP t), or -1
template <int CMP>
__device__ int64_t t_bytes_find(const uint8_t *fbase, int64_t a, int64_t b, uint32_t t) {
    constexpr bool MAX = (CMP == CMP_GT || CMP == CMP_GEQ);
    const uintptr_t fb = reinterpret_cast<uintptr_t>(fbase);
    for (uintptr_t ga = (fb + (uintptr_t)a) & ~(uintptr_t)15; ga < fb + (uintptr_t)b; ga += 16) {
        int64_t pos0;
        const uint4 v = t_granule<MAX>(fbase, ga, a, b, pos0);
        if (!cmp_holds<CMP>(vext16<MAX>(v), t)) continue;
        for (int j = 0; j < 16; ++j) {
            const int64_t pos = pos0 + j;
            if (pos >= a && pos < b && cmp_holds<CMP>(vbyte(v, j), t)) return pos;
        }
    }
    return -1;
}
template <int ALGO>
__device__ int64_t t_step_bytes(const uint8_t *fbase, int64_t x, int64_t w, int64_t mx, int64_t Lf) {
    const int64_t limit = Lf - x < mx ? Lf : x + mx;
    if constexpr (ALGO == ALGO_RAM) {
        if (x + w >= Lf) return Lf;  // the window does not fit: a single final chunk
        const uint32_t M = t_bytes_ext<true>(fbase, x, x + w);
        const int64_t i = x + w < limit ? t_bytes_find<CMP_GEQ>(fbase, x + w, limit, M) : -1;
        return i >= 0 ? i + 1 : limit;
    } else {
        constexpr bool MAX = ALGO == ALGO_AE_MAX;
        constexpr int CMP = MAX ? CMP_GT : CMP_LT;
        int64_t t = x;
        uint32_t v = fbase[x];
        while (t + w < limit) {
            const int64_t r = t_bytes_find<CMP>(fbase, t + 1, t + w + 1, v);
            if (r < 0) return t + w + 1;  // the target is unbeaten over its window
            t = r;
            v = fbase[r];
        }
        return limit;
    }
}
// one chunk step: from the index when it decides the step, else from the
// bytes while the chain's budget of byte steps lasts (a lane reads up to a
// window per byte step; long unsaturated stretches, such as large zero-filled
// regions, are left to the speculative walk): -1 when the budget is spent
#ifndef CDC_T_BYTE_STEPS
#define CDC_T_BYTE_STEPS 4
#endif
constexpr int T_BYTE_STEPS = CDC_T_BYTE_STEPS;
template <int ALGO>
__device__ __forceinline__ int64_t t_next(const uint8_t *fbase, const uint32_t *ix, uint32_t n, int64_t lo,
                                          int64_t ihi, int64_t x, int64_t w, int64_t mx, int64_t Lf, int &budget) {
    const int64_t y = t_step<ALGO>(ix, n, lo, ihi, x, w, mx, Lf);
    if (y >= 0) return y;
    // inside a constant run (value c) both rules end the chunk at x+w+1: RAM's
    // window maximum is c and d[x+w] = c; AE's target c is unbeaten over (x, x+w]
    const uint32_t *runs = ix + T_IX_CAP;
    const int64_t limit = Lf - x < mx ? Lf : x + mx;
    for (uint32_t r = 0; r < runs[0]; ++r) {
        const int64_t rs = lo + (int64_t)runs[1 + 3 * r], re = lo + (int64_t)runs[2 + 3 * r];
        if (x >= rs && x + w < re && x + w + 1 <= limit) return x + w + 1;
    }
    if (--budget < 0) return -1;
    return t_step_bytes<ALGO>(fbase, x, w, mx, Lf);
}

// candidates of segment [pa, ...): index range [*i0, *i0 + K) of their
// saturating positions (K = 0: none, a segment inside a long constant run);
// T_UNKNOWN when the index [lo, ihi) does not decide the set.  Segments g-1
// and g compute the set of g from different indexes and must agree on it (the
// rows of g's extra entries follow its candidates), so "not in my index"
// never reads as "none".
constexpr uint32_t T_UNKNOWN = 0xFFFFFFFFu;
template <int ALGO>
__device__ __forceinline__ uint32_t t_cands(const uint32_t *ix, uint32_t n, int64_t lo, int64_t ihi, int64_t Lf,
                                            int64_t pa, int64_t w, uint32_t &i0) {
    int64_t clo = ALGO == ALGO_RAM ? pa - 1 : pa - w - 1;  // lowest candidate position
    const int64_t chi = ALGO == ALGO_RAM ? pa + w - 1 : pa - 1;  // the last is N(chi)
    if (clo < 0) clo = 0;
    if (clo < lo) return T_UNKNOWN;
    i0 = t_lb(ix, n, (uint32_t)(clo - lo));
    const uint32_t i1 = t_lb(ix, n, (uint32_t)(chi - lo));
    if (i1 < n) return i1 - i0 + 1;
    return ihi >= Lf ? n - i0 : T_UNKNOWN;  // N(chi) past the stream end: every later one
}
// upper end of a segment's index.  A chain's last step inside the segment
// starts before seg_end: AE reads its target range (x, x + w] only, RAM the
// first saturating byte at or after x + w, which uniform-like bytes put a few
// hundred bytes later; RAM's candidates of the next segment reach N(seg_end
// + w - 1).  So the index stops 4 KiB (AE) or 16 KiB (RAM: room for short
// unsaturated stretches there) past seg_end + w, not at seg_end + max_size:
// a step that would need more is read from the bytes, a candidate set it
// cannot decide makes the attempt fall back.  ~12 % (AE) / ~8 % (RAM) less
// index work at the default caps.
template <int ALGO>
__device__ __forceinline__ int64_t t_ihi(int64_t seg_end, int64_t w, int64_t mx, int64_t Lf) {
    int64_t h = seg_end + w + (ALGO == ALGO_RAM ? 16384 : 4096);
    if (ALGO != ALGO_RAM && h > seg_end + mx + 1) h = seg_end + mx + 1;  // AE never reads past the cap
    return h < Lf ? h : Lf;
}
__device__ __forceinline__ int64_t t_start_of(int algo, int64_t satpos, int64_t w) {
    return algo == ALGO_RAM ? satpos + 1 : satpos + w + 1;
}

// start of candidate k of segment g (segment 0's only candidate is the
// stream start)
template <int ALGO>
__device__ __forceinline__ int64_t t_cand_start(uint64_t g, const uint32_t *ix, int64_t lo, uint32_t c0, uint32_t k,
                                                int64_t w) {
    return g == 0 ? 0 : t_start_of(ALGO, lo + (int64_t)ix[c0 + k], w);
}

// link of a chain that exits segment g at x: the index of x among the
// candidates of g+1 (d0 .. d0+KN-1 in the index), T_END at the stream end, or
// T_BAD when x is not a candidate
template <int ALGO>
__device__ __forceinline__ uint32_t t_link(const uint32_t *ix, uint32_t n, int64_t lo, int64_t x, int64_t w,
                                           int64_t Lf, bool last, uint32_t d0, uint32_t KN) {
    if (last) return x >= Lf ? T_END : T_BAD;
    const int64_t satpos = ALGO == ALGO_RAM ? x - 1 : x - w - 1;
    if (satpos < lo) return T_BAD;
    const uint32_t i = t_lb(ix, n, (uint32_t)(satpos - lo));
    return (i < n && lo + (int64_t)ix[i] == satpos && i >= d0 && i < d0 + KN) ? i - d0 : T_BAD;
}

// Transfer table of segment g, phase 1: the rows of its candidates (W.tl,
// W.tn).  A chain whose exit is not a candidate of g+1 (its last step was not
// saturated) becomes an extra entry of g+1: its start goes to W.tex[g] and
// its link to KN + j; the count is published in W.tnx[g] for phase 2 of g+1.
// Returns K (the candidates; -1 when the segment cannot be resolved in index
// space).
template <int ALGO>
__device__ int t_table(const Geometry &G, Work &W, uint64_t g, const SegInfo &I, const uint8_t *fbase,
                       const uint32_t *ix, uint32_t n, int64_t lo, int64_t ihi, uint32_t *pos) {
    const int lane = lane_id();
    const int64_t w = G.w, mx = (int64_t)G.max_size, Lf = (int64_t)I.Lf;
    uint32_t c0 = 0;
    // no candidates (a segment that starts in a long constant run): every
    // entry then comes as an extra entry from segment g-1
    const uint32_t K = g == 0 ? 1u : t_cands<ALGO>(ix, n, lo, ihi, Lf, I.p, w, c0);
    uint32_t d0 = 0, KN = 0;
    const bool last = g == I.last;
    if (!last) KN = t_cands<ALGO>(ix, n, lo, ihi, Lf, I.seg_end, w, d0);
    if (K > (uint32_t)TK || KN > (uint32_t)TK) {
        if (lane == 0) st_release_u32(W.tnx + g, 0u);
        return -1;
    }
    uint32_t nx = 0;  // extra entries passed on so far
    for (uint32_t k0 = 0; k0 < K; k0 += 32) {
        const uint32_t k = k0 + lane;
        int64_t x = -1;
        uint32_t cnt = 0;
        if (k < K) {
            x = t_cand_start<ALGO>(g, ix, lo, c0, k, w);
            int budget = T_BYTE_STEPS;
            while (x >= 0 && x < I.seg_end) {
                if (pos && cnt < (uint32_t)TPOS) pos[cnt * TK + k] = (uint32_t)(x - I.p);
                ++cnt;
                x = t_next<ALGO>(fbase, ix, n, lo, ihi, x, w, mx, Lf, budget);
            }
        }
        uint32_t link = k < K && x >= 0 ? t_link<ALGO>(ix, n, lo, x, w, Lf, last, d0, KN) : T_BAD;
        const bool extra = k < K && x >= 0 && link == T_BAD && !last;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, extra);
        if (extra) {
            const uint32_t j = nx + __popc(bal & ((1u << lane) - 1u));
            if (j < (uint32_t)TEX && KN + j < (uint32_t)TK) {
                W.tex[g * TEX + j] = x;
                link = KN + j;
            }
#ifdef CDC_T_CONST_SAMPLE
            else atomicAdd(W.ctrl + 10, j >= (uint32_t)TEX ? 1u : 0x10000u);  // (experiment) which limit
#endif
        }
#ifdef CDC_T_CONST_SAMPLE
        if (k < K && x >= 0 && link == T_BAD && last) atomicAdd(W.ctrl + 10, 0x1000000u);
#endif
        nx += __popc(bal);
        if (k < K && link == T_BAD) atomicAdd(W.ctrl + (x < 0 ? 14 : 15), 1u);  // diagnostics: budget / overflow
        if (k < K) {
            W.tl[g * TK + k] = link;
            W.tn[g * TK + k] = cnt;
        }
    }
    __syncwarp();
    if (lane == 0) {
        __threadfence();
        st_release_u32(W.tnx + g, nx < (uint32_t)TEX ? nx : (uint32_t)TEX);
    }
    return (int)K;
}

// Phase 2: the rows of the extra entries segment g-1 passed on (rows K ..
// K+X-1).  Their exits must be candidates of g+1 or exits this segment's
// phase 1 already handed over (no new hand-over).
template <int ALGO>
__device__ bool t_table_extras(const Geometry &G, Work &W, uint64_t g, const SegInfo &I, const uint8_t *fbase,
                               const uint32_t *ix, uint32_t n, int64_t lo, int64_t ihi, uint32_t K, uint32_t *pos) {
    const int lane = lane_id();
    const int64_t w = G.w, mx = (int64_t)G.max_size, Lf = (int64_t)I.Lf;
    uint32_t X = 0;
    if (g > 0) {
        if (lane == 0) {
            const unsigned long long t0 = globaltimer();
            uint32_t ns = 64;
            for (;;) {
                X = ld_acquire_u32(W.tnx + g - 1);
                if (X != ~0u) break;
                if (!t_alive(W) || globaltimer() - t0 > T_TIMEOUT_NS) {
                    X = ~0u;
                    break;
                }
                __nanosleep(ns);
                if (ns < 1024) ns <<= 1;
            }
        }
        X = __shfl_sync(0xFFFFFFFFu, X, 0);
        if (X == ~0u || K + X > (uint32_t)TK) return false;
    }
    uint32_t d0 = 0, KN = 0;
    const bool last = g == I.last;
    if (!last) KN = t_cands<ALGO>(ix, n, lo, ihi, Lf, I.seg_end, w, d0);
    for (uint32_t j = lane; j < X; j += 32) {
        int64_t x = W.tex[(g - 1) * TEX + j];
        uint32_t cnt = 0;
        int budget = T_BYTE_STEPS;
        while (x >= 0 && x < I.seg_end) {
            if (pos && cnt < (uint32_t)TPOS) pos[cnt * TK + K + j] = (uint32_t)(x - I.p);
            ++cnt;
            x = t_next<ALGO>(fbase, ix, n, lo, ihi, x, w, mx, Lf, budget);
        }
        uint32_t lk = x >= 0 ? t_link<ALGO>(ix, n, lo, x, w, Lf, last, d0, KN) : T_BAD;
        if (lk == T_BAD && x >= 0 && !last) {
            // an exit this segment's own candidate chains hand over already (the
            // chains met before the boundary): the same extra entry of g+1
            const uint32_t nxo = ld_relaxed_u32(W.tnx + g);
            for (uint32_t q = 0; q < nxo && q < (uint32_t)TEX; ++q)
                if (W.tex[g * TEX + q] == x && KN + q < (uint32_t)TK) {
                    lk = KN + q;
                    break;
                }
        }
        if (lk == T_BAD) atomicAdd(W.ctrl + (x < 0 ? 14 : 11), 1u);  // diagnostics: budget / second hand-over
        W.tl[g * TK + K + j] = lk;
        W.tn[g * TK + K + j] = cnt;
    }
    if (lane == 0) W.tk[g] = K + X;
    return true;
}

// Segments form blocks of TB: block b holds [TB b, min(TB (b+1), nsegs)).
constexpr int TB = 32;
__device__ __forceinline__ uint64_t t_blk_lo(uint64_t b) { return b * TB; }

// gather: entry `idx` (0..TK) of a row held 4 per lane (entry u*32 + lane in r[u])
__device__ __forceinline__ uint32_t t_gather(const uint32_t (&r)[4], uint32_t idx) {
    const int src = (int)(idx & 31u);
    const uint32_t v0 = __shfl_sync(0xFFFFFFFFu, r[0], src), v1 = __shfl_sync(0xFFFFFFFFu, r[1], src);
    const uint32_t v2 = __shfl_sync(0xFFFFFFFFu, r[2], src), v3 = __shfl_sync(0xFFFFFFFFu, r[3], src);
    const uint32_t u = idx >> 5;
    return u == 0 ? v0 : u == 1 ? v1 : u == 2 ? v2 : v3;
}

// Compose block b's tables (the last of its walkers to publish does this):
// for every entry candidate k of its first segment, the entry candidate and
// the chain starts before each member (W.tp, W.tq), and the block's link and
// start count (W.tbc, W.tbs).  Rows load four members at a time, so the
// shuffle chain waits for one L2 round trip per four members.
__device__ void t_compose(Work &W, uint64_t b, uint64_t nsegs) {
    const int lane = lane_id();
    const uint64_t hs = t_blk_lo(b), he = (b + 1) * TB < nsegs ? (b + 1) * TB : nsegs;
    // narrow tables (every member has at most 64 rows, the common case): two
    // rows per lane, eight members per L2 round trip
    const uint32_t myk = lane < (int)(he - hs) ? W.tk[hs + lane] : 0u;
    if (__reduce_max_sync(0xFFFFFFFFu, myk) <= 64u) {
        constexpr int HB = 8;  // members per L2 round trip
        const uint32_t K0 = __shfl_sync(0xFFFFFFFFu, myk, 0);
        uint32_t c2[2], a2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint32_t k = (uint32_t)(u * 32 + lane);
            c2[u] = k < K0 ? k : T_BAD;
            a2[u] = 0;
        }
        for (int v0 = 0; v0 < TB; v0 += HB) {
            uint32_t L2[HB][2], N2[HB][2];
#pragma unroll
            for (int v = 0; v < HB; ++v) {
                const uint64_t h = hs + v0 + v;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    L2[v][u] = h < he ? W.tl[h * TK + u * 32 + lane] : T_BAD;
                    N2[v][u] = h < he ? W.tn[h * TK + u * 32 + lane] : 0u;
                }
            }
#pragma unroll
            for (int v = 0; v < HB; ++v) {
                const uint64_t h = hs + v0 + v;
                const uint32_t Kh = __shfl_sync(0xFFFFFFFFu, myk, v0 + v);
                if (h < he) {  // uniform across the warp
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        W.tp[h * TK + u * 32 + lane] = c2[u];
                        W.tq[h * TK + u * 32 + lane] = a2[u];
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const bool in = h < he && c2[u] < Kh;
                    const uint32_t idx = in ? c2[u] : 0u;
                    const int src = (int)(idx & 31u);
                    const uint32_t l0 = __shfl_sync(0xFFFFFFFFu, L2[v][0], src);
                    const uint32_t l1 = __shfl_sync(0xFFFFFFFFu, L2[v][1], src);
                    const uint32_t n0 = __shfl_sync(0xFFFFFFFFu, N2[v][0], src);
                    const uint32_t n1 = __shfl_sync(0xFFFFFFFFu, N2[v][1], src);
                    if (h < he) {
                        a2[u] += in ? (idx >> 5 ? n1 : n0) : 0u;
                        c2[u] = in ? (idx >> 5 ? l1 : l0) : T_BAD;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            W.tbc[b * TK + u * 32 + lane] = u < 2 ? c2[u & 1] : T_BAD;
            W.tbs[b * TK + u * 32 + lane] = u < 2 ? a2[u & 1] : 0u;
        }
        return;
    }
    const uint32_t K0 = W.tk[hs];
    uint32_t cur[4], acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint32_t k = (uint32_t)(u * 32 + lane);
        cur[u] = k < K0 ? k : T_BAD;
        acc[u] = 0;
    }
    for (uint64_t h0 = hs; h0 < he; h0 += 4) {
        uint32_t L[4][4], N[4][4], Kh[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint64_t h = h0 + v;
            Kh[v] = h < he ? W.tk[h] : 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                L[v][u] = h < he ? W.tl[h * TK + u * 32 + lane] : T_BAD;
                N[v][u] = h < he ? W.tn[h * TK + u * 32 + lane] : 0u;
            }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint64_t h = h0 + v;
            if (h >= he) break;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                W.tp[h * TK + u * 32 + lane] = cur[u];
                W.tq[h * TK + u * 32 + lane] = acc[u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool in = cur[u] < Kh[v];
                const uint32_t idx = in ? cur[u] : 0u;
                const uint32_t l = t_gather(L[v], idx), n = t_gather(N[v], idx);
                acc[u] += in ? n : 0u;
                cur[u] = in ? l : T_BAD;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        W.tbc[b * TK + u * 32 + lane] = cur[u];
        W.tbs[b * TK + u * 32 + lane] = acc[u];
    }
}

// The scan over blocks (the last composer does it): the true chain starts
// at segment 0's only candidate.  Rows load ahead of the shuffle chain.
// False when some block cannot continue the chain.
__device__ bool t_scan_blocks(Work &W, uint64_t nsegs, uint64_t *d_count) {
    const int lane = lane_id();
    const uint64_t NB = (nsegs + TB - 1) / TB;
    uint32_t E = 0;
    uint64_t O = 0;
    for (uint64_t b0 = 0; b0 < NB; b0 += 4) {  // four blocks' rows per L2 round trip
        uint32_t C[4][4], S[4][4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                C[v][u] = b0 + v < NB ? W.tbc[(b0 + v) * TK + u * 32 + lane] : T_BAD;
                S[v][u] = b0 + v < NB ? W.tbs[(b0 + v) * TK + u * 32 + lane] : 0u;
            }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint64_t b = b0 + v;
            if (b >= NB) break;
            if (E >= (uint32_t)TK) {
                if (lane == 0) t_fail(W, E == T_END ? 9 : 7, b * TB);
                return false;
            }
            if (lane == 0) {
                W.tbe[b] = E;
                W.tbo[b] = O;
            }
            const uint32_t c = t_gather(C[v], E), sc = t_gather(S[v], E);
            if (c == T_BAD) {
                if (lane == 0) t_fail(W, 8, b * TB);
                return false;
            }
            O += sc;
            E = c;
        }
    }
    if (E != T_END) {
        if (lane == 0) t_fail(W, 11, nsegs);
        return false;
    }
    if (lane == 0) {
        W.seg_out[nsegs] = O;
        *d_count = O;
    }
    return true;
}

// One T-mode attempt of walker g, before any byte walk (all 32 lanes).
// Returns true when the call's output was produced from the tables (this
// walker has written its part); false to fall back to the speculative walk.
template <int ALGO>
__device__ bool t_attempt(const Geometry &G, Work &W, uint64_t g, uint64_t nsegs, const SegInfo &I,
                          uint8_t *ring, const uint8_t *fbase, uint64_t *bounds, uint64_t cap, uint64_t *d_count,
                          int64_t pre_n) {
    constexpr bool MAX = ALGO != ALGO_AE_MIN;
    const int lane = lane_id();
    const int64_t w = G.w, mx = (int64_t)G.max_size, Lf = (int64_t)I.Lf;
    uint32_t *ix = reinterpret_cast<uint32_t *>(ring);
    uint32_t *pos = pre_n >= 0 ? reinterpret_cast<uint32_t *>(ring + RING_SMEM) : nullptr;
    const int64_t lo = I.p - w - 1 > 0 ? I.p - w - 1 : 0;
    const int64_t ihi = t_ihi<ALGO>(I.seg_end, w, mx, Lf);
    unsigned long long *tm = g_timing ? g_timing + TM_STAMPS + TM_PER_SEG * g : nullptr;
    uint32_t n = 0;
    if (pre_n >= 0) {  // the CTA built the index together (t_coop_index)
        n = (uint32_t)pre_n;
        bool mine = t_alive(W) && n <= T_IX_CAP &&
                    (uint64_t)n * (uint64_t)(w + 1) >= (uint64_t)T_DENSE * (uint64_t)(ihi - lo);
        const int K = mine ? t_table<ALGO>(G, W, g, I, fbase, ix, n, lo, ihi, pos) : -1;
        mine = K >= 0 && t_table_extras<ALGO>(G, W, g, I, fbase, ix, n, lo, ihi, (uint32_t)K, pos);
        if (tm && lane == 0) tm[6] = globaltimer();
        if (!mine) t_fail(W);
    } else if (t_alive(W)) {
        // a cheap look at the segment's first 16 KiB first: clearly sparse, no
        // index (half the density the full check asks for: uniform bytes at
        // w = 8 KiB give 64 +- 8 saturating bytes there, the bar is 8)
        const int64_t shi = I.p + 16384 < ihi ? I.p + 16384 : ihi;
        const uint32_t ns = t_index<MAX>(fbase, I.p, shi, I.p, ix, T_IDX_CAP);
        bool mine = 2ull * ns * (uint64_t)(w + 1) >= (uint64_t)T_DENSE * (uint64_t)(shi - I.p);
#ifdef CDC_T_CONST_SAMPLE
        mine = mine || t_constant(fbase, I.p, shi);
#endif
        uint32_t why = 1;
        if (mine) {
            n = t_index<MAX>(fbase, lo, ihi, lo, ix, T_IX_CAP, W.ctrl + T_ALL, ix + T_IX_CAP);
            t_buckets(ix, n, ihi - lo);
            if (tm && lane == 0) tm[5] = globaltimer();
            // a long constant run (a zero-filled region, say): its chains keep their
            // phases, too many to hand over; the speculative walk is the better path
#ifdef CDC_T_CONST_SAMPLE
            uint64_t span = (uint64_t)(ihi - lo);  // (experiment) density outside the constant runs
            for (uint32_t r = 0; r < ix[T_IX_CAP]; ++r)
                span -= (uint64_t)(ix[T_IX_CAP + 2 + 3 * r] - ix[T_IX_CAP + 1 + 3 * r]);
#else
            const uint64_t span = (uint64_t)(ihi - lo);
#endif
            why = n == T_IX_CAP + 2 ? 4 : n > T_IX_CAP ? 2
                : (uint64_t)n * (uint64_t)(w + 1) < (uint64_t)T_DENSE * span ? 3
                : ix[T_IX_CAP + 1 + 3 * TRUNS] >= T_LONG_RUN ? 4 : 0;
            const int K = why == 0 ? t_table<ALGO>(G, W, g, I, fbase, ix, n, lo, ihi, pos) : -1;
            if (why == 0 && K < 0) why = 5;
            if (why == 0 && !t_table_extras<ALGO>(G, W, g, I, fbase, ix, n, lo, ihi, (uint32_t)K, pos)) why = 6;
            mine = why == 0;
            if (tm && lane == 0) tm[6] = globaltimer();
        }
        if (!mine && lane == 0) t_fail(W, why, g);
        __syncwarp();
    }
    // arrive: the last walker of a block composes the block, the last composer
    // scans the blocks.  The verdict word T_SCAN decides once (compare-and-
    // swap from ~0): 1 = the tables produced the output, 0 = fall back.
    const uint64_t NB = (nsegs + TB - 1) / TB;
    const uint64_t b = g / TB;
    const uint64_t members = ((b + 1) * TB < nsegs ? (b + 1) * TB : nsegs) - t_blk_lo(b);
    bool composer = false, scanner = false;
    __syncwarp();
    if (lane == 0) {
        if (tm) tm[2] = globaltimer();  // diagnostics: table published
        __threadfence();
        composer = atomicAdd(W.tblk + b, 1u) + 2u == (uint32_t)members;  // starts at ~0
    }
    composer = __shfl_sync(0xFFFFFFFFu, composer, 0);
    if (composer) {
        __threadfence();
        if (t_alive(W)) t_compose(W, b, nsegs);
        __syncwarp();
        if (lane == 0) {
            if (tm) tm[4] = globaltimer();  // diagnostics: block composed
            __threadfence();
            scanner = atomicAdd(W.ctrl + T_ARRIVE, 1u) + 2u == (uint32_t)NB;
        }
    }
    scanner = __shfl_sync(0xFFFFFFFFu, scanner, 0);
    if (scanner) {  // every block composed
        __threadfence();
        bool ok = t_alive(W) && nsegs >= 2;
        if (ok) ok = t_scan_blocks(W, nsegs, d_count);
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicCAS(W.ctrl + T_SCAN, ~0u, ok ? 1u : 0u);
            if (tm) tm[5] = globaltimer();  // diagnostics: scan done (replaces the index stamp)
        }
    }
    uint32_t verdict = 0;
    if (lane == 0) {
        const unsigned long long t0 = globaltimer();
        uint32_t ns = 64;
        for (;;) {
            verdict = ld_acquire_u32(W.ctrl + T_SCAN);
            if (verdict != ~0u) break;
            if (!t_alive(W) || globaltimer() - t0 > T_TIMEOUT_NS) {
                if (t_alive(W)) t_fail(W, 10, g);
                atomicCAS(W.ctrl + T_SCAN, ~0u, 0u);  // give up (unless the scan has just decided)
                continue;
            }
            __nanosleep(ns);
            if (ns < 1024) ns <<= 1;
        }
    }
    verdict = __shfl_sync(0xFFFFFFFFu, verdict, 0);
    if (tm && lane == 0) tm[1] = globaltimer();  // diagnostics: verdict seen
    if (verdict != 1u) return false;
    // this segment's part of the true chain: copied from the chain-start store
    // when the table pass kept it, else walked again in index space by lane 0
    const uint32_t Eb = W.tbe[b];
    const uint32_t E = W.tp[g * TK + Eb];
    const uint64_t q0 = W.tbo[b] + W.tq[g * TK + Eb];
    const uint32_t cntE = W.tn[g * TK + E];
    if (pos && cntE <= (uint32_t)TPOS) {
        for (uint32_t j = lane; j < cntE; j += 32) {
            const uint64_t q = q0 + j;
            if (q >= 1 && q - 1 < cap) bounds[q - 1] = (uint64_t)I.p + pos[j * TK + E];  // the stream start is not a boundary
        }
    } else if (lane == 0) {
        uint64_t q = q0;
        uint32_t c0 = 0;
        const uint32_t Kc = g == 0 ? 1u : t_cands<ALGO>(ix, n, lo, ihi, Lf, I.p, w, c0);
        // a candidate, or an extra entry handed over by segment g-1
        int64_t x = E < Kc ? t_cand_start<ALGO>(g, ix, lo, c0, E, w) : W.tex[(g - 1) * TEX + (E - Kc)];
        int budget = 1 << 30;  // the scan followed this chain: its table row was resolved
        while (x < I.seg_end) {
            if (q >= 1 && q - 1 < cap) bounds[q - 1] = (uint64_t)x;
            ++q;
            x = t_next<ALGO>(fbase, ix, n, lo, ihi, x, w, mx, Lf, budget);
        }
    }
    if (lane == 0 && g == nsegs - 1) {
        const uint64_t total = W.seg_out[nsegs];
        if (total >= 1 && total - 1 < cap) bounds[total - 1] = (uint64_t)Lf;  // the last boundary is the length
    }
    return true;
}

// T-mode, one segment per CTA (a small stream): the CTA's 16 warps index the
// saturating bytes of [p - w - 1, t_ihi) together, one
// sixteenth each into their own rings, and warp 0 concatenates the parts in
// order into its ring.  Returns the entry count for warp 0 (T_IX_CAP + 1:
// not dense or too many), or -1 when the attempt is already off.  All threads
// of the CTA call this.
template <int ALGO>
__device__ int64_t t_coop_index(const Geometry &G, Work &W, uint64_t g, uint8_t *rings) {
    constexpr bool MAX = ALGO != ALGO_AE_MIN;
    __shared__ uint32_t s_cnt[SPEC_WARPS];
    __shared__ int s_go;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const SegInfo I = seg_info(G, W, g);
    const uint8_t *fbase = G.data + I.foff;
    const int64_t w = G.w, Lf = (int64_t)I.Lf;
    const int64_t lo = I.p - w - 1 > 0 ? I.p - w - 1 : 0;
    const int64_t ihi = t_ihi<ALGO>(I.seg_end, w, (int64_t)G.max_size, Lf);
    uint32_t *ix = reinterpret_cast<uint32_t *>(rings + warp * RING_SMEM);
    // the density sample of t_attempt (the segment's first 16 KiB), one
    // sixteenth per warp
    const int64_t shi = I.p + 16384 < ihi ? I.p + 16384 : ihi;
    {
        const int64_t sp = (((shi - I.p) + 16 * SPEC_WARPS - 1) / (16 * SPEC_WARPS)) * 16;
        const int64_t sa = I.p + warp * sp, sb = sa + sp < shi ? sa + sp : shi;
        const uint32_t c = sa < sb ? t_index<MAX>(fbase, sa, sb, sa, ix, T_IDX_CAP) : 0u;
        if (lane == 0) s_cnt[warp] = c;
    }
    __syncthreads();
    if (warp == 0) {
        int go = 0;
        if (t_alive(W)) {
            uint64_t ns = 0;
            for (int k = 0; k < SPEC_WARPS; ++k) ns += s_cnt[k];
            go = 2ull * ns * (uint64_t)(w + 1) >= (uint64_t)T_DENSE * (uint64_t)(shi - I.p) ? 1 : 2;
        }
        if (lane == 0) s_go = go;
    }
    __syncthreads();
    const int go = s_go;
    if (go == 0) return -1;
    if (go == 1) {
        const int64_t part = (((ihi - lo) + 16 * SPEC_WARPS - 1) / (16 * SPEC_WARPS)) * 16;
        const int64_t a = lo + warp * part, b = a + part < ihi ? a + part : ihi;
        const uint32_t c = a < b ? t_index<MAX>(fbase, a, b, lo, ix, T_IX_CAP) : 0u;
        if (lane == 0) s_cnt[warp] = c;
    }
    __syncthreads();
    if (go == 2) {
        if (warp == 0 && lane == 0) t_fail(W, 1, g);
        return (int64_t)T_IX_CAP + 1;
    }
    if (warp != 0) return 0;  // only warp 0 walks the segment
    if (lane == 0) ix[T_IX_CAP] = 0;  // no constant runs recorded on this path (its samples reject them)
    uint32_t n = 0;
    for (int k = 0; k < SPEC_WARPS; ++k) {
        const uint32_t c = s_cnt[k];
        if (c > T_IX_CAP || n + c > T_IX_CAP) return (int64_t)T_IX_CAP + 1;
        if (k > 0) {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(rings + k * RING_SMEM);
            for (uint32_t i = lane; i < c; i += 32) ix[n + i] = src[i];
        }
        n += c;
    }
    __syncwarp();
    t_buckets(ix, n, ihi - lo);
    return (int64_t)n;
}

