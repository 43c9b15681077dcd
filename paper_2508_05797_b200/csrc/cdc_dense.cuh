// cdc_dense.cuh -- dense-index mode: a small single stream whose every window
// holds the saturating byte (included by cdc_kernels.cu inside namespace cdc;
// DESIGN.md §6 "Dense-index mode").
//
// On such a stream both rules reduce to one recurrence over the positions
// P[0] < P[1] < ... of the saturating byte (0xFF for RAM and AE-Max, 0x00 for
// AE-Min):
//   RAM (§2.1.2 l.198): the window [s, s+w) holds a saturating byte, so its
//     maximum is saturated and the chunk ends after the first saturating byte
//     b >= s+w: e = b+1; the next chunk's boundary byte is the first
//     saturating byte >= b + w + 1.
//   AE (l.169): the first saturating byte q of [s, s+w] is a target no byte
//     beats, and every earlier target is beaten within w bytes, so e = q+w+1;
//     the next chunk's q is the first saturating byte >= q + w + 1.
// So the chain is x_0, x_{k+1} = first P >= x_k + w + 1, with x_0 = first
// P >= w (RAM) or first P >= 0 (AE), and the chunk ends are x_k + 1 (RAM) or
// x_k + w + 1 (AE), clamped to the stream length L, followed by L itself when
// the last one falls short of it.  This holds for every start the chain can
// reach when   P[0] <= w-1,  P[i+1] - P[i] <= w  for all i,  L-1 - P[last] <= w
// (every interval of w bytes then holds a saturating byte, the stream's tail
// after the last one is a final chunk (R7)) and max_size >= 2w+2 (no chunk
// reaches the cap: reading R5).  The kernels check exactly that condition and
// give the call to the ordinary pipeline (its gate) when it fails.
//
// k_dense_index  one CTA per segment of ~L/#SMs bytes (persistent over
//   segments): the sorted positions of the saturating bytes of the segment and
//   of the 2w bytes after it (coalesced 16-byte loads, eight 512-byte blocks in
//   flight per warp, exact per-byte masks, ballot ranks), a 256-byte bucket
//   table for lookups, and the segment's transfer table: the chain enters the
//   segment at one of its candidates -- the positions in [p_g, p_g + w) and the
//   first one at or after p_g + w -- and thread r follows candidate r through
//   the segment, recording its elements (rows) and publishing (exit candidate
//   of the next segment, element count).  No CTA ever waits for another.
// k_dense_resolve  one CTA (PDL behind the index kernel) loads every table into
//   shared memory, follows the true chain through the segments in three short
//   passes and writes each segment's entry row and output offset, and the gate.
// k_dense_finish  one warp per segment copies the entry row's elements to the
//   output as chunk ends (or, when the gate opened, resets the ordinary
//   pipeline's lists).
#pragma once

constexpr int DN_THREADS = 768;
constexpr int DN_WARPS = DN_THREADS / 32;
constexpr int DN_NV = 11;           // 512-byte blocks a warp keeps in flight (a 128 KiB region in one round)
constexpr int DN_WCAP = 128;        // saturating positions per warp's share of a segment's region
constexpr int DN_ICAP = 4096;       // ... per segment region
constexpr int DN_CAND = 128;        // candidates (table rows) per segment
constexpr int DN_BKT = 1536;        // 256-byte buckets per segment region
constexpr int DN_GMAX = 1024;       // segments
constexpr uint32_t DN_END = 0xFFFFu;
constexpr uint32_t DN_SMAX = 128u << 10, DN_SMIN = 64u << 10;  // segment bytes
constexpr uint32_t DN_WMAX = 24u << 10;                         // largest window
constexpr int DN_SMEM = 150 << 10;  // dynamic shared memory of k_dense_index
constexpr int DN_TCAP = (DN_SMEM - 8 * (DN_GMAX + 1) - 8 * DN_WARPS * DN_CAND - 64) / 4;  // table entries the resolver holds
constexpr uint32_t DN_BAD = 0xFFFEu;  // (resolver) a row that is no candidate of its segment

struct DGeo {
    const uint8_t *data;
    uint64_t L;
    uint32_t G, S;      // segments [g S, (g+1) S), the last one up to L
    uint32_t w;
    uint32_t steps;     // capacity of a row (elements of one candidate's chain inside a segment)
    uint32_t ext;       // bytes indexed past a segment's end
    int ram;            // 1 RAM, 0 AE
    int max;            // 1: the saturating byte is 0xFF, 0: 0x00
};
struct DWork {
    unsigned long long *ctrl;  // [0] the call's abort word: DN_ABORT once a segment gave up (any other value: none
                        // did, so a fresh workspace needs no reset); k_dense_resolve leaves 0
    uint32_t *gate;     // written by the last CTA: 0 = the output is written here, 1 = run the ordinary pipeline
    uint32_t *nc;       // G: candidates per segment; nc[G]: the entry row of segment 0
    uint32_t *tab;      // G x DN_CAND: exit row << 16 | elements
    uint32_t *rows;     // G x DN_CAND x steps: element positions relative to the segment start
    uint64_t *ent;      // G: entry row | output offset << 32 (~0: the chain ended before the segment)
};

constexpr unsigned long long DN_ABORT = 0x9E3779B97F4A7C15ull;
__device__ __forceinline__ void dn_fail(const DWork &X) { *reinterpret_cast<volatile unsigned long long *>(X.ctrl) = DN_ABORT; }
__device__ __forceinline__ bool dn_aborted(const DWork &X) { return __ldcg(X.ctrl) == DN_ABORT; }
// diagnostic stamps (cdc_debug_timing, tools/dense_timing.py): per segment {start, index built,
// checked + buckets, table published}; after the G segments {resolve begin, tables loaded, done, pass 1, pass 2}
__device__ __forceinline__ void dn_stamp(uint32_t g, int k) {
    unsigned long long *tm = g_timing;
    if (tm != nullptr && threadIdx.x == 0) tm[TM_STAMPS + (uint64_t)TM_PER_SEG * g + k] = globaltimer();
}

// does the 16-byte vector hold the saturating byte?  (the zero-byte test of (x - 0x01010101) & ~x &
// 0x80808080, on ~x for 0xFF: nonzero iff some byte is zero; two operations per word)
template <bool MAX>
__device__ __forceinline__ bool dn_any_sat(const uint4 &v) {
    auto z = [](uint32_t x) -> uint32_t {
        return MAX ? ((~x - 0x01010101u) & x & 0x80808080u) : ((x - 0x01010101u) & ~x & 0x80808080u);
    };
    return (z(v.x) | z(v.y) | z(v.z) | z(v.w)) != 0u;
}

template <bool MAX>
__device__ __forceinline__ void dn_segment(const DGeo &Q, const DWork &X, uint32_t g, uint8_t *smem) {
    uint32_t *wl = reinterpret_cast<uint32_t *>(smem);                  // DN_WARPS x DN_WCAP
    uint32_t *pos = wl + DN_WARPS * DN_WCAP;                            // DN_ICAP (+1)
    uint16_t *succ = reinterpret_cast<uint16_t *>(pos + DN_ICAP + 4);   // DN_ICAP: index of the next chain element
    uint16_t *bkt = succ + DN_ICAP;                                      // DN_BKT
    __shared__ uint32_t s_wc[DN_WARPS + 1];
    __shared__ uint32_t s_bad;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p = (int64_t)g * Q.S;
    const int64_t pe = g + 1 == Q.G ? (int64_t)Q.L : p + Q.S;
    const int64_t hi = min((int64_t)Q.L, pe + (int64_t)Q.ext);
    const uint32_t Sg = (uint32_t)(pe - p), R = (uint32_t)(hi - p);  // segment and region lengths
    // 16-byte granules of the region, from the aligned address at or below its first byte
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(Q.data + p);
    const uint32_t mis = (uint32_t)(a0 & 15u);
    const uint4 *gran = reinterpret_cast<const uint4 *>(a0 - mis);
    const uint32_t ng = (R + mis + 15u) / 16u;
    const uint32_t nblk = (ng + 31u) / 32u, bpw = (nblk + DN_WARPS - 1) / DN_WARPS;
    if (threadIdx.x == 0) s_bad = 0;
    dn_stamp(g, 0);
    // ---- the warp's share: blocks [b0, b1) of 32 granules, DN_NV in flight
    uint32_t wc = 0;
    const uint32_t b0 = min(nblk, (uint32_t)warp * bpw), b1 = min(nblk, b0 + bpw);
    uint32_t *mine = wl + warp * DN_WCAP;
    for (uint32_t b = b0; b < b1; b += DN_NV) {
        uint4 v[DN_NV];
#pragma unroll
        for (int k = 0; k < DN_NV; ++k) {
            const uint32_t gi = (b + k) * 32u + (uint32_t)lane;
            v[k] = (b + k < b1 && gi < ng) ? __ldcs(gran + gi) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < DN_NV; ++k) {
            const uint32_t gi = (b + k) * 32u + (uint32_t)lane;
            const int q = (int)(gi * 16u) - (int)mis;  // region-relative position of the granule's first byte
            const bool any = b + k < b1 && gi < ng && dn_any_sat<MAX>(v[k]);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, any);
            if (k == 0 && b == b0) dn_stamp(g, 5);
            if (bal == 0u) continue;
            uint32_t m = 0;
            if (any) {
                m = sat_mask16<MAX>(v[k]);
                if (q < 0 || q + 16 > (int)R) {  // (the region's first and last granule)
                    const int ka = min(max(-q, 0), 16), kb = min(max((int)R - q, 0), 16);
                    m &= ((1u << kb) - 1u) & ~((1u << ka) - 1u);
                }
            }
            const uint32_t c = (uint32_t)__popc(m);
            uint32_t rank, tot;
            if (__ballot_sync(0xFFFFFFFFu, any && c != 1u) == 0u) {  // one per granule that holds any
                rank = (uint32_t)__popc(bal & ((1u << lane) - 1u));
                tot = (uint32_t)__popc(bal);
            } else {
                uint32_t inc = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                    if (lane >= d) inc += t;
                }
                rank = inc - c;
                tot = __shfl_sync(0xFFFFFFFFu, inc, 31);
            }
            if (wc + tot > (uint32_t)DN_WCAP) {
                wc = 0xFFFF0000u;  // (overflow: far too many saturating bytes for this mode)
                break;
            }
            uint32_t mm = m, o = wc + rank;
            while (mm) {
                const int bit = __ffs(mm) - 1;
                mm &= mm - 1u;
                mine[o++] = (uint32_t)(q + bit);
            }
            wc += tot;
        }
        if (wc >= 0xFFFF0000u) break;
    }
    dn_stamp(g, 6);
    if (lane == 0) s_wc[warp] = wc;
    __syncthreads();
    // ---- compact the warps' lists into pos[0, n)
    uint32_t base = 0, n = 0;
    bool over = false;
    for (int j = 0; j < DN_WARPS; ++j) {
        const uint32_t c = s_wc[j];
        over |= c >= 0xFFFF0000u;
        if (j < warp) base += c;
        n += c;
    }
    if (over || n > (uint32_t)DN_ICAP || n == 0u || R / 256u + 2u > (uint32_t)DN_BKT) {
        if (threadIdx.x == 0) dn_fail(X);
        return;
    }
    for (uint32_t i = lane; i < wc; i += 32) pos[base + i] = mine[i];
    __syncthreads();
    dn_stamp(g, 1);
    // ---- the density condition on this segment's positions, and the bucket table
    const uint32_t nb = R / 256u + 1u;  // buckets 0..nb (bkt[k]: first index with pos >= 256 k)
    bool bad = false;
    for (uint32_t i = threadIdx.x; i <= n; i += DN_THREADS) {
        const uint32_t x = i < n ? pos[i] : 0u;
        const uint32_t k0 = i == 0 ? 0u : (pos[i - 1] >> 8) + 1u;
        const uint32_t k1 = i < n ? (x >> 8) : nb;
        for (uint32_t k = k0; k <= k1 && k <= nb; ++k) bkt[k] = (uint16_t)i;
        if (i < n && x < Sg) {
            if (i + 1 < n) bad |= pos[i + 1] - x > Q.w;
            else bad |= !(hi == (int64_t)Q.L && (uint32_t)(Q.L - 1 - (uint64_t)(p + x)) <= Q.w);
        }
        if (i == 0 && g == 0) bad |= x > Q.w - 1u;
    }
    if (bad) s_bad = 1;
    __syncthreads();
    if (s_bad) {
        if (threadIdx.x == 0) dn_fail(X);
        return;
    }
    dn_stamp(g, 2);
    auto lower = [&](uint32_t t) -> uint32_t {  // first index with pos >= t
        const uint32_t k = t >> 8;
        if (k > nb) return n;
        uint32_t i = bkt[k];
        while (i < n && pos[i] < t) ++i;
        return i;
    };
    // ---- candidates and their chains through the segment
    const uint32_t iw = lower(Q.w), ncand = min(iw + 1u, n), iend = lower(Sg);
    if (ncand > (uint32_t)DN_CAND) {
        if (threadIdx.x == 0) dn_fail(X);
        return;
    }
    // every position's successor in the chain, all at once; a row then only chases indices
    for (uint32_t i = threadIdx.x; i < iend; i += DN_THREADS) succ[i] = (uint16_t)lower(pos[i] + Q.w + 1u);
    __syncthreads();
    if (threadIdx.x < ncand) {
        const uint32_t r = threadIdx.x;
        uint32_t *row = X.rows + ((uint64_t)g * DN_CAND + r) * Q.steps;
        uint32_t i = r, cnt = 0, ex = DN_END;
        bool ok = true;
        for (;;) {
            if (i >= iend) {  // the first element past the segment
                ex = i - iend;
                break;
            }
            if (cnt >= Q.steps) {
                ok = false;
                break;
            }
            row[cnt++] = pos[i];
            i = succ[i];
            if (i >= n) {
                ok = hi == (int64_t)Q.L;  // the chain ends with the stream
                ex = DN_END;
                break;
            }
        }
        if (!ok || (ex != DN_END && ex >= (uint32_t)DN_CAND)) dn_fail(X);
        X.tab[(uint64_t)g * DN_CAND + r] = (ex << 16) | cnt;
    }
    if (threadIdx.x == 0) {
        X.nc[g] = ncand;
        if (g == 0) {
            X.nc[Q.G] = Q.ram ? iw : 0u;       // x_0: the first position >= w (RAM) or >= 0 (AE)
            if (Q.ram && iw >= n) dn_fail(X);
        }
    }
}

// The true chain through the segments (k_dense_resolve's one CTA):
// every table in shared memory, then three short passes instead of one walk
// over all G segments -- warp b takes the block of BS consecutive segments
// [b BS, (b+1) BS) and follows every candidate of its first segment through the
// block (exit row, elements); one thread follows the true entry through the
// DN_WARPS blocks; each warp follows its block's true entry again and writes
// the segments' entries.
__device__ __forceinline__ void dn_resolve(const DGeo &Q, const DWork &X, uint8_t *smem) {
    uint32_t *toff = reinterpret_cast<uint32_t *>(smem);  // G + 1: where segment g's table starts in stab
    uint32_t *tcnt = toff + DN_GMAX + 1;                   // G: its rows
    uint32_t *bex = tcnt + DN_GMAX + 1;                    // DN_WARPS x DN_CAND: a block's exit row per entry row
    uint32_t *bacc = bex + DN_WARPS * DN_CAND;             // ... and its elements
    uint32_t *stab = bacc + DN_WARPS * DN_CAND;            // the tables
    __shared__ uint32_t s_tot, s_fail;
    __shared__ uint32_t s_brow[DN_WARPS];
    __shared__ uint32_t s_boff[DN_WARPS];
    const uint32_t G = Q.G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    dn_stamp(G, 0);
    __shared__ uint32_t s_r0;
    if (threadIdx.x == 0) {
        s_fail = 0;
        s_r0 = __ldcg(X.nc + G);  // the entry row of segment 0
    }
    if (threadIdx.x < DN_WARPS) s_brow[threadIdx.x] = DN_END;
    const bool gave_up = dn_aborted(X);  // (read along with the tables)
    bool fail = false;
    if (G * (uint32_t)DN_CAND <= (uint32_t)DN_TCAP) {
        // few segments: every table at a fixed stride of DN_CAND rows, so the table loads need not wait
        // for the candidate counts (rows past a segment's count are never looked at): one round trip
        for (uint32_t g = threadIdx.x; g < G; g += DN_THREADS) {
            tcnt[g] = min(__ldcg(X.nc + g), (uint32_t)DN_CAND);
            toff[g] = g * DN_CAND;
        }
        for (uint32_t j0 = warp; j0 < G; j0 += DN_WARPS * 4) {
            uint32_t v[4][DN_CAND / 32], c[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const uint32_t g = j0 + a * DN_WARPS;
                c[a] = g < G ? __ldcg(X.nc + g) : 0u;
#pragma unroll
                for (int q = 0; q < DN_CAND / 32; ++q)
                    v[a][q] = g < G ? __ldcg(X.tab + (uint64_t)g * DN_CAND + lane + 32 * q) : 0u;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {  // (rows past the segment's count: never written, marked as no candidates)
                const uint32_t g = j0 + a * DN_WARPS;
#pragma unroll
                for (int q = 0; q < DN_CAND / 32; ++q)
                    if (g < G) stab[g * DN_CAND + lane + 32 * q] = (uint32_t)(lane + 32 * q) < c[a] ? v[a][q] : DN_BAD << 16;
            }
        }
        fail = gave_up;
    } else {
        for (uint32_t g = threadIdx.x; g < G; g += DN_THREADS) tcnt[g] = min(__ldcg(X.nc + g), (uint32_t)DN_CAND);
        __syncthreads();
        if (threadIdx.x < 32) {  // exclusive prefix of the candidate counts: toff[g] = entries before segment g
            uint32_t run = 0;
            for (uint32_t g0 = 0; g0 < G; g0 += 32) {
                const uint32_t g = g0 + threadIdx.x;
                const uint32_t c = g < G ? tcnt[g] : 0u;
                uint32_t inc = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                    if ((int)threadIdx.x >= d) inc += t;
                }
                if (g < G) toff[g] = run + inc - c;
                run += __shfl_sync(0xFFFFFFFFu, inc, 31);
            }
            if (threadIdx.x == 0) s_tot = run;
        }
        __syncthreads();
        fail = gave_up || s_tot > (uint32_t)DN_TCAP;
        if (!fail) {  // the tables, packed: four segments' loads in flight per warp
            for (uint32_t j0 = warp; j0 < G; j0 += DN_WARPS * 4) {
                uint32_t v[4][DN_CAND / 32];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const uint32_t g = j0 + a * DN_WARPS;
                    const uint32_t c = g < G ? tcnt[g] : 0u;
#pragma unroll
                    for (int q = 0; q < DN_CAND / 32; ++q) {
                        const uint32_t r = lane + 32 * q;
                        v[a][q] = r < c ? __ldcg(X.tab + (uint64_t)g * DN_CAND + r) : 0u;
                    }
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const uint32_t g = j0 + a * DN_WARPS;
                    const uint32_t c = g < G ? tcnt[g] : 0u;
#pragma unroll
                    for (int q = 0; q < DN_CAND / 32; ++q) {
                        const uint32_t r = lane + 32 * q;
                        if (r < c) stab[toff[g] + r] = v[a][q];
                    }
                }
            }
        }
    }
    __syncthreads();
    dn_stamp(G, 1);
    const bool stride = G * (uint32_t)DN_CAND <= (uint32_t)DN_TCAP;
    const uint32_t BS = (G + DN_WARPS - 1) / DN_WARPS;
    const uint32_t g0 = min(G, (uint32_t)warp * BS), g1 = min(G, g0 + BS);
    if (!fail && g0 < g1) {  // pass 1: every row of the block's first segment through the block, four per lane
        uint32_t row[DN_CAND / 32], acc[DN_CAND / 32];
        const uint32_t c0 = tcnt[g0];
#pragma unroll
        for (int q = 0; q < DN_CAND / 32; ++q) {
            row[q] = (uint32_t)(lane + 32 * q) < c0 ? (uint32_t)(lane + 32 * q) : DN_BAD;
            acc[q] = 0;
        }
        for (uint32_t g = g0; g < g1; ++g) {
            const uint32_t lim = stride ? (uint32_t)DN_CAND : tcnt[g], o = toff[g];
#pragma unroll
            for (int q = 0; q < DN_CAND / 32; ++q) {
                if (row[q] < lim) {
                    const uint32_t t = stab[o + row[q]];
                    acc[q] += t & 0xFFFFu;
                    row[q] = t >> 16;
                } else if (row[q] < DN_BAD) {
                    row[q] = DN_BAD;  // (packed tables: a row that is no candidate of this segment)
                }
            }
        }
#pragma unroll
        for (int q = 0; q < DN_CAND / 32; ++q) {
            bex[warp * DN_CAND + lane + 32 * q] = row[q];
            bacc[warp * DN_CAND + lane + 32 * q] = acc[q];
        }
    }
    __syncthreads();
    dn_stamp(G, 3);
    if (threadIdx.x == 0 && !fail) {  // pass 2: the true chain, block by block
        uint32_t row = s_r0, off = 0;
        const int nblk = (int)((G + BS - 1) / BS);
        for (int b = 0; b < nblk; ++b) {
            s_brow[b] = row;
            s_boff[b] = off;
            if (row >= (uint32_t)DN_CAND) break;  // DN_END: the chain ended; DN_BAD: give up
            off += bacc[b * DN_CAND + row];
            row = bex[b * DN_CAND + row];
        }
        if (row != DN_END) s_fail = 1;  // (the last segment's chains all end with the stream)
    }
    dn_stamp(G, 4);
    __syncthreads();
    if (lane == 0 && !fail && !s_fail && g0 < g1) {  // pass 3: the segments' entries
        uint32_t row = s_brow[warp];
        unsigned long long off = s_boff[warp];
        uint32_t g = g0;
        for (; g < g1 && row < (uint32_t)DN_CAND; ++g) {
            X.ent[g] = (uint64_t)row | (off << 32);
            const uint32_t t = stab[toff[g] + row];
            off += t & 0xFFFFu;
            row = t >> 16;
        }
        for (; g < g1; ++g) X.ent[g] = ~0ull;  // the chain ended before these
    }
    if (threadIdx.x == 0) {
        *X.gate = (fail || s_fail) ? 1u : 0u;
        dn_stamp(G, 2);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(DN_THREADS, 1) k_dense_index(DGeo Q, DWork X) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t s_go;
    pdl_trigger();  // (k_dense_resolve waits for this grid's completion before it reads anything)
    for (uint32_t g = blockIdx.x; g < Q.G; g += gridDim.x) {
        if (threadIdx.x == 0) s_go = dn_aborted(X) ? 0u : 1u;
        __syncthreads();
        if (s_go) {  // (else another segment gave up: nothing left to do)
            if (Q.max) dn_segment<true>(Q, X, g, smem);
            else dn_segment<false>(Q, X, g, smem);
        }
        dn_stamp(g, 3);
        __syncthreads();
    }
}

// One CTA, launched with PDL behind k_dense_index: the true chain through the
// segments' tables, each segment's entry row and output offset, the gate.
__global__ void __launch_bounds__(DN_THREADS, 1) k_dense_resolve(DGeo Q, DWork X) {
    extern __shared__ __align__(128) uint8_t smem[];
    pdl_wait();
    pdl_trigger();
    dn_resolve(Q, X, smem);
    if (threadIdx.x == 0) *X.ctrl = 0ull;  // (after every thread's read of it: dn_resolve ends with barriers)
}

// After k_dense_index: when its gate is shut, one warp per segment copies the
// entry row's elements to the output as chunk ends; when it is open, this is
// the ordinary pipeline's list reset (k_reset's loop over [p, p + n16)), so the
// fallback costs no extra launch and the dense path none for the reset.
__global__ void __launch_bounds__(256) k_dense_finish(DGeo Q, DWork X, uint64_t *bounds, uint64_t cap, uint64_t *d_count,
                                                      uint4 *rst, uint64_t n16) {
    pdl_wait();
    pdl_trigger();
    if (*X.gate != 0u) {
        const uint4 ones = make_uint4(~0u, ~0u, ~0u, ~0u);
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
            rst[i] = ones;
        return;
    }
    const int lane = threadIdx.x & 31;
    const uint32_t g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (g >= Q.G) return;
    const uint64_t e = X.ent[g];
    if (e == ~0ull) return;
    const uint32_t row = (uint32_t)e;
    const uint64_t off = e >> 32;
    const uint32_t t = X.tab[(uint64_t)g * DN_CAND + row];
    const uint32_t cnt = t & 0xFFFFu;
    const uint32_t *rw = X.rows + ((uint64_t)g * DN_CAND + row) * Q.steps;
    const uint64_t p = (uint64_t)g * Q.S, delta = Q.ram ? 1ull : (uint64_t)Q.w + 1ull;
    for (uint32_t k = lane; k < cnt; k += 32) {
        const uint64_t x = min(p + rw[k] + delta, Q.L);
        if (off + k < cap) bounds[off + k] = x;
    }
    if ((t >> 16) == DN_END && lane == 0) {  // the chain's last element: the stream's last chunk ends at L
        const uint64_t last = cnt ? min(p + rw[cnt - 1] + delta, Q.L) : 0ull;
        uint64_t total = off + cnt;
        if (last < Q.L) {
            if (total < cap) bounds[total] = Q.L;
            ++total;
        }
        *d_count = total;
    }
}
