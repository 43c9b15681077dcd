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
//   of the next segment, element count).  The CTA that draws the last ticket
//   loads every table into shared memory, follows the true chain through the
//   segments (one lookup per segment) and writes each segment's entry row and
//   output offset: no CTA ever waits for another.
// k_dense_write  one warp per segment copies the entry row's elements to the
//   output as chunk ends.
#pragma once

constexpr int DN_THREADS = 512;
constexpr int DN_WARPS = DN_THREADS / 32;
constexpr int DN_WCAP = 256;        // saturating positions per warp's share of a segment's region
constexpr int DN_ICAP = 4096;       // ... per segment region
constexpr int DN_CAND = 128;        // candidates (table rows) per segment
constexpr int DN_BKT = 1536;        // 256-byte buckets per segment region
constexpr int DN_GMAX = 1024;       // segments
constexpr uint32_t DN_END = 0xFFFFu;
constexpr uint32_t DN_SMAX = 128u << 10, DN_SMIN = 64u << 10;  // segment bytes
constexpr uint32_t DN_WMAX = 24u << 10;                         // largest window
constexpr int DN_SMEM = 150 << 10;  // dynamic shared memory of k_dense_index
constexpr int DN_TCAP = (DN_SMEM - 4 * (DN_GMAX + 1) - 64) / 4;  // table entries the resolver holds

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
    uint32_t *ctrl;     // [0] segment ticket, [1] failure flag (reset to ~0 by k_reset)
    uint32_t *gate;     // written by the last CTA: 0 = the output is written here, 1 = run the ordinary pipeline
    uint32_t *nc;       // G: candidates per segment; nc[G]: the entry row of segment 0
    uint32_t *tab;      // G x DN_CAND: exit row << 16 | elements
    uint32_t *rows;     // G x DN_CAND x steps: element positions relative to the segment start
    uint64_t *ent;      // G: entry row | output offset << 32 (~0: the chain ended before the segment)
};

__device__ __forceinline__ void dn_fail(const DWork &X) { atomicExch(X.ctrl + 1, 0u); }

template <bool MAX>
__device__ void dn_segment(const DGeo &Q, const DWork &X, uint32_t g, uint8_t *smem) {
    uint32_t *wl = reinterpret_cast<uint32_t *>(smem);                  // DN_WARPS x DN_WCAP
    uint32_t *pos = wl + DN_WARPS * DN_WCAP;                            // DN_ICAP (+1)
    uint16_t *bkt = reinterpret_cast<uint16_t *>(pos + DN_ICAP + 4);    // DN_BKT
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
    // ---- the warp's share: blocks [b0, b1) of 32 granules, eight in flight
    uint32_t wc = 0;
    const uint32_t b0 = min(nblk, (uint32_t)warp * bpw), b1 = min(nblk, b0 + bpw);
    uint32_t *mine = wl + warp * DN_WCAP;
    for (uint32_t b = b0; b < b1; b += 8) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t gi = (b + k) * 32u + (uint32_t)lane;
            v[k] = (b + k < b1 && gi < ng) ? __ldcs(gran + gi) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t gi = (b + k) * 32u + (uint32_t)lane;
            const int q = (int)(gi * 16u) - (int)mis;  // region-relative position of the granule's first byte
            uint32_t m = 0;
            if (b + k < b1 && gi < ng) {
                const int ka = min(max(-q, 0), 16), kb = min(max((int)R - q, 0), 16);
                m = sat_mask16<MAX>(v[k]) & ((1u << kb) - 1u) & ~((1u << ka) - 1u);
            }
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m != 0u);
            if (bal == 0u) continue;
            const uint32_t c = (uint32_t)__popc(m);
            uint32_t rank, tot;
            if (__ballot_sync(0xFFFFFFFFu, c > 1u) == 0u) {  // at most one per granule
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
    if (threadIdx.x < ncand) {
        const uint32_t r = threadIdx.x;
        uint32_t *row = X.rows + ((uint64_t)g * DN_CAND + r) * Q.steps;
        uint32_t i = r, cnt = 0, ex = DN_END;
        bool ok = true;
        for (;;) {
            const uint32_t x = pos[i];
            if (x >= Sg) {
                ex = i - iend;
                break;
            }
            if (cnt >= Q.steps) {
                ok = false;
                break;
            }
            row[cnt++] = x;
            i = lower(x + Q.w + 1u);
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

// The true chain through the segments (the CTA that drew the last ticket).
__device__ void dn_resolve(const DGeo &Q, const DWork &X, uint8_t *smem) {
    uint32_t *toff = reinterpret_cast<uint32_t *>(smem);  // G + 1
    uint32_t *stab = toff + DN_GMAX + 1;                   // the tables, packed
    __shared__ uint32_t s_tot;
    const uint32_t G = Q.G;
    for (uint32_t g = threadIdx.x; g < G; g += DN_THREADS) toff[g + 1] = min(__ldcg(X.nc + g), (uint32_t)DN_CAND);
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive prefix of the candidate counts: toff[g] = entries before segment g
        uint32_t run = 0;
        for (uint32_t g0 = 0; g0 < G; g0 += 32) {
            const uint32_t g = g0 + threadIdx.x;
            const uint32_t c = g < G ? toff[g + 1] : 0u;
            uint32_t inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if ((int)threadIdx.x >= d) inc += t;
            }
            __syncwarp();
            if (g < G) toff[g + 1] = run + inc;
            run += __shfl_sync(0xFFFFFFFFu, inc, 31);
        }
        if (threadIdx.x == 0) {
            toff[0] = 0;
            s_tot = run;
        }
    }
    __syncthreads();
    bool fail = __ldcg(X.ctrl + 1) != 0xFFFFFFFFu || s_tot > (uint32_t)DN_TCAP;
    if (!fail) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (uint32_t g = warp; g < G; g += DN_WARPS) {
            const uint32_t c = toff[g + 1] - toff[g];
            for (uint32_t r = lane; r < c; r += 32) stab[toff[g] + r] = __ldcg(X.tab + (uint64_t)g * DN_CAND + r);
        }
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (!fail) {
        uint32_t row = __ldcg(X.nc + G);
        uint64_t off = 0;
        uint32_t g = 0;
        for (; g < G; ++g) {
            if (row >= toff[g + 1] - toff[g]) {
                fail = true;
                break;
            }
            X.ent[g] = (uint64_t)row | (off << 32);
            const uint32_t t = stab[toff[g] + row];
            off += t & 0xFFFFu;
            row = t >> 16;
            if (row == DN_END) break;
        }
        if (g == G) fail = true;  // (the last segment's chains all end with the stream)
        for (++g; g < G; ++g) X.ent[g] = ~0ull;
        if (off >= (1ull << 32)) fail = true;
    }
    *X.gate = fail ? 1u : 0u;
}

__global__ void __launch_bounds__(DN_THREADS, 1) k_dense_index(DGeo Q, DWork X) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t s_last, s_go;
    pdl_wait();     // the reset of ctrl has completed
    pdl_trigger();
    for (uint32_t g = blockIdx.x; g < Q.G; g += gridDim.x) {
        if (threadIdx.x == 0) s_go = __ldcg(X.ctrl + 1) == 0xFFFFFFFFu ? 1u : 0u;
        __syncthreads();
        if (s_go) {  // (else another segment gave up: only the tickets are left to take)
            if (Q.max) dn_segment<true>(Q, X, g, smem);
            else dn_segment<false>(Q, X, g, smem);
        }
        __threadfence();  // this segment's table and rows before its ticket
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(X.ctrl, 1u) + 1u == Q.G - 1u ? 1u : 0u;  // the counter starts at ~0
        __syncthreads();
        if (s_last) {
            __threadfence();
            dn_resolve(Q, X, smem);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_dense_write(DGeo Q, DWork X, uint64_t *bounds, uint64_t cap, uint64_t *d_count) {
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const uint32_t g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (g >= Q.G || *X.gate != 0u) return;
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
