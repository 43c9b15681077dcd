// cdc_maxp.cuh -- MAXP on sm_100a (§2.1.2 l.173 and l.196, §4.3 l.361).
//
// MAXP ends a chunk right after a target byte that is greater than the h bytes
// before it and the h bytes after it ("the target byte's value is greater than
// the maximum value from both windows", l.196; readings M1-M4 in DESIGN.md §2).
// Whether a byte is such a local maximum does not depend on where chunks
// start, so the GPU form splits the method in two ("MAXP"):
//
//  1. k_maxp_scan (HBM-bound, one pass over the bytes): every tile of MX_TILE
//     candidate positions is copied with its two h-byte margins into shared
//     memory by one TMA bulk copy; the local maxima of the tile are found with
//     Extreme Byte Searches over 16-byte granules (§4.1: one max per granule,
//     then one per block of MX_BG granules by shuffles).  A local maximum is
//     its block's maximum and beats the NBK blocks on each side that lie
//     wholly inside its windows, so only blocks that pass this filter (a few
//     percent on uniform bytes) get the exact test: one warp checks the
//     K0 whole granules on each side and the window bytes beyond them.  Each tile writes its maxima to its
//     own slot (no tile waits for another); k_maxp_gather then concatenates
//     the slots in stream order (a scan of the tile counts) into one
//     ascending list of elements: per file, a virtual "file start" element
//     followed by the file's maxima (file-relative positions).
//  0. (k_maxp_files) A batch: tiles never cross files; every file gets
//     max(1, ceil(len / MX_TILE)) tiles, the tile table comes from a scan of
//     those counts.  A single stream is a batch of one file.
//  2. The chain (what depends on chunk starts): from a start s the chunk ends
//     after the first local maximum in [s+h, s+max_size) (M3, R5), else it is
//     capped.  Two local maxima are more than h apart, so after a content
//     boundary at q[i] the next one is q[i+1] unless the gap exceeds max_size;
//     only capped stretches can skip a maximum (one that falls within h of a
//     cap start).  k_maxp_link computes for every element i (and the stream
//     start, i = -1) where its chunk run ends, f(i), and its cap count;
//     k_maxp_path walks the (rare) runs that skip maxima, in order, and marks
//     the skipped ones; k_maxp_write scans the per-element boundary counts
//     (decoupled look-back) and writes caps and content boundaries.
//
// Nothing here is shared with oracle/ (tests compare the two element by element).
// (Included by cdc_kernels.cu inside namespace cdc.)

#ifndef CDC_MX_TILE
#define CDC_MX_TILE 32768
#endif
constexpr int MX_TILE = CDC_MX_TILE;   // candidate positions per scan tile
constexpr int MX_THREADS = 256;        // k_maxp_scan
constexpr uint32_t MX_HMAX = 65536;    // largest window per side a tile's shared memory holds
constexpr int MX_ETILE = 256;          // elements per link / write tile (one thread each)
constexpr int MX_GTILES = 1024;        // scan tiles per k_maxp_gather CTA (one thread each)
constexpr int MX_BG = 8;               // granules per block of k_maxp_scan's block filter (lanes per shuffle group)

struct MaxpGeo {
    const uint8_t *data;
    const uint64_t *file_off;  // batch: nfiles+1 file offsets into data; null: one stream of L bytes
    uint64_t nfiles;
    uint64_t L, h, M;      // stream (or batch) length, window per side, max_size
    uint64_t ntiles;       // scan tiles (an upper bound for a batch: the files' count is on the device)
    uint64_t qcap;         // element capacity (L / (h+1) + 2 nfiles + 2: local maxima are > h apart)
    uint32_t buf;          // bytes of a tile's byte buffer in shared memory
    uint32_t ccap;         // candidates per tile (uint16 offsets)
};
struct MaxpWork {
    uint64_t *tfirst;            // nfiles+1: first scan tile of each file (the last: the tile count)
    uint32_t *tfile;             // file of each scan tile
    uint16_t *qt;                // scan tile t's maxima (offsets from the tile start): [t * ccap, ...)
    uint32_t *qn;                // ... and their number
    int64_t *qx;                 // elements: a file's start (-1), then its maxima (file-relative), file by file
    uint32_t *efile;             // file of each element
    uint64_t *estart;            // nfiles+1: each file's start element (the last: the element count)
    int64_t *f;                  // element e: the element where e's chunk run ends (estart[file+1]: the file end)
    uint64_t *ncap;              // ... and the number of capped chunks in that run
    int64_t *jl;                 // elements whose run skips a local maximum, ascending
    uint64_t *bo;                // batch: nfiles+1 output offsets of each file's boundaries (null: one stream)
    // reset to ~0 (all-ones) before every call:
    unsigned long long *fst;     // file-table CTAs' look-back words
    unsigned long long *tst;     // gather CTAs' look-back words
    unsigned long long *lst;     // link tiles' look-back words
    unsigned long long *wst;     // write tiles' look-back words
    uint32_t *ctrl;              // tickets: [0] scan, [1] link, [2] write, [3] gather, [4] file table
    unsigned long long *nq;      // number of elements (written by the last gather CTA)
    unsigned long long *nj;      // number of skipping runs (last link tile)
    uint8_t *on;                 // element e: 0xFF on the chain, 0 skipped
};

__device__ __forceinline__ void mx_file(const MaxpGeo &Q, uint64_t F, uint64_t &off, uint64_t &len) {
    if (Q.file_off == nullptr) {
        off = 0;
        len = Q.L;
    } else {
        off = Q.file_off[F];
        len = Q.file_off[F + 1] - off;
    }
}

// byte-wise maximum of a 16-byte granule (four 4-way byte maxima, then the word's bytes)
__device__ __forceinline__ uint32_t granule_max(const uint4 &v) {
    uint32_t m = __vmaxu4(__vmaxu4(v.x, v.y), __vmaxu4(v.z, v.w));
    m = __vmaxu4(m, m >> 16);
    m = __vmaxu4(m, m >> 8);
    return m & 0xFFu;
}

// block-wide exclusive scan of one 32-bit value per thread (MX_THREADS or 1024 threads)
__device__ __forceinline__ uint32_t mx_block_scan(uint32_t v, uint32_t &total, uint32_t *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = lane < nw ? scratch[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= o) s += y;
        }
        scratch[32 + lane] = s;
    }
    __syncthreads();
    const uint32_t before = warp ? scratch[32 + warp - 1] : 0u;
    total = scratch[32 + nw - 1];
    __syncthreads();
    return before + x - v;
}

// Tile t's exclusive prefix of a count, published as TL_AGG then TL_INC
// (warp 0; the result is returned to every thread through `slot`).
__device__ __forceinline__ uint64_t mx_tile_prefix(unsigned long long *st, uint64_t t, uint64_t cnt, uint64_t *slot) {
    if (threadIdx.x < 32) {
        uint64_t excl = 0;
        if (t == 0) {
            if (threadIdx.x == 0) tile_publish(st, TL_INC, cnt);
        } else {
            if (threadIdx.x == 0) tile_publish(st + t, TL_AGG, cnt);
            excl = tile_lookback(st, 1, t);
            if (threadIdx.x == 0) tile_publish(st + t, TL_INC, excl + cnt);
        }
        if (threadIdx.x == 0) *slot = excl;
    }
    __syncthreads();
    const uint64_t r = *slot;
    __syncthreads();
    return r;
}

constexpr int MX_FTHREADS = 1024;  // k_maxp_files: files per CTA (one thread each)
// K0: the tile table: file F owns tiles [tfirst[F], tfirst[F+1]), max(1, ceil(len/MX_TILE))
// of them (an empty file keeps one, so that every file has a start element).
__global__ void __launch_bounds__(MX_FTHREADS) k_maxp_files(MaxpGeo Q, MaxpWork X) {
    __shared__ uint32_t s_tile, s_scr[64];
    __shared__ uint64_t s_slot;
    if (threadIdx.x == 0) s_tile = atomicAdd(X.ctrl + 4, 1u) + 1u;
    __syncthreads();
    const uint64_t g = s_tile;
    const uint64_t F = g * MX_FTHREADS + threadIdx.x;
    uint32_t n = 0;
    uint64_t off = 0, len = 0;
    if (F < Q.nfiles) {
        mx_file(Q, F, off, len);
        n = len == 0 ? 1u : (uint32_t)((len + MX_TILE - 1) / MX_TILE);
    }
    uint32_t tot;
    const uint32_t o = mx_block_scan(n, tot, s_scr);
    const uint64_t excl = mx_tile_prefix(X.fst, g, tot, &s_slot);
    if (F < Q.nfiles) X.tfirst[F] = excl + o;
    // tile -> file map (a single stream has none: its scan and gather know the file is 0); each
    // warp writes its 32 files' tiles with all lanes, so one large file is not one thread's loop
    if (Q.file_off != nullptr) {
        const int lane = threadIdx.x & 31;
        for (int r = 0; r < 32; ++r) {
            const uint32_t rn = __shfl_sync(0xFFFFFFFFu, n, r);
            const uint64_t rt = __shfl_sync(0xFFFFFFFFu, excl + o, r);
            const uint32_t rF = __shfl_sync(0xFFFFFFFFu, (uint32_t)F, r);
            for (uint32_t k = lane; k < rn; k += 32) X.tfile[rt + k] = rF;
        }
    }
    if ((g + 1) * MX_FTHREADS >= Q.nfiles && threadIdx.x == 0) X.tfirst[Q.nfiles] = excl + tot;
}

// K1: local maxima, tile by tile (static schedule, the next tile prefetched into L2).
__global__ void __launch_bounds__(MX_THREADS) k_maxp_scan(MaxpGeo Q, MaxpWork X) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t s_scr[64], s_cnt, s_ns;
    uint8_t *buf = align_smem(smem);                       // tile bytes (Q.buf)
    uint8_t *gm = buf + Q.buf;                             // granule maxima
    const uint32_t NGmax = Q.buf / 16;
    const uint32_t NBmax = NGmax / MX_BG + 1;
    uint8_t *bm = gm + NGmax;                              // block maxima (MX_BG granules)
    uint16_t *surv = reinterpret_cast<uint16_t *>(bm + ((NBmax + 1) & ~1u));  // blocks (granules) that pass the filter
    uint16_t *cand = surv + NGmax / 2 + 1;
    const int tid = threadIdx.x;
    const uint64_t h = Q.h;
    const uint64_t ntot = X.tfirst[Q.nfiles];
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    // the tile's file and its candidate positions [ca, cb) inside [h, L - h) (file-relative;
    // a single stream skips the table lookups)
    auto tile_range = [&](uint64_t t, uint64_t &foff, uint64_t &L, uint64_t &a, uint64_t &ca, uint64_t &cb) {
        foff = 0;
        L = Q.L;
        a = t * MX_TILE;
        if (Q.file_off != nullptr) {
            const uint32_t F = X.tfile[t];
            mx_file(Q, F, foff, L);
            a = (t - X.tfirst[F]) * MX_TILE;
        }
        const uint64_t b = a + MX_TILE < L ? a + MX_TILE : L;
        ca = a > h ? a : h;
        cb = (L > h && b > L - h) ? L - h : (L > h ? b : 0);
    };
    // tiles blockIdx.x, + gridDim.x, ... (one wave of CTAs); while a tile is copied and
    // scanned, its CTA's next tile is already being fetched into L2 (one bulk prefetch)
#ifndef CDC_MX_PF
#define CDC_MX_PF 0
#endif
#ifndef CDC_MX_STATIC
#define CDC_MX_STATIC 0
#endif
    __shared__ uint32_t s_tile;
    for (uint64_t t = blockIdx.x;; t += gridDim.x) {
        if (!CDC_MX_STATIC) {
            if (tid == 0) s_tile = atomicAdd(X.ctrl, 1u) + 1u;  // the counter starts at ~0
            __syncthreads();
            t = s_tile;
        }
        if (t >= ntot) break;
        if (CDC_MX_PF && tid == 0 && t + gridDim.x < ntot) {
            uint64_t pfo, pL, pa, pca, pcb;
            tile_range(t + gridDim.x, pfo, pL, pa, pca, pcb);
            if (pca < pcb) {
                const uintptr_t p0 = reinterpret_cast<uintptr_t>(Q.data + pfo + (pca - h)) & ~static_cast<uintptr_t>(15);
                const uintptr_t p1 = (reinterpret_cast<uintptr_t>(Q.data + pfo + (pcb + h)) + 15) & ~static_cast<uintptr_t>(15);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"((uint32_t)(p1 - p0)) : "memory");
            }
        }
        uint64_t foff, L, a, ca, cb;
        tile_range(t, foff, L, a, ca, cb);
        const uint8_t *data = Q.data + foff;
        uint32_t count = 0;
        bool ranked = false;  // the long-window path writes its slot itself
        if (tid == 0) s_cnt = s_ns = 0;
        if (ca < cb) {
            // bytes [lo, hi) = [ca - h, cb + h): one bulk copy of the 16-byte granules holding them
            const uint64_t lo = ca - h, hi = cb + h;
            const uintptr_t A0 = reinterpret_cast<uintptr_t>(data + lo) & ~static_cast<uintptr_t>(15);
            const uintptr_t A1 = (reinterpret_cast<uintptr_t>(data + hi) + 15) & ~static_cast<uintptr_t>(15);
            const uint32_t nbytes = (uint32_t)(A1 - A0);
            const uint32_t off0 = (uint32_t)(reinterpret_cast<uintptr_t>(data + lo) - A0);
            if (tid == 0) {
                mbar_arrive_expect_tx(&bar, nbytes);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_addr(buf)),
                    "l"(reinterpret_cast<const uint8_t *>(A0)), "r"(nbytes), "r"(smem_addr(&bar))
                    : "memory");
            }
            mbar_wait(&bar, phase);
            phase ^= 1u;
            // bytes of the first and last granule outside [lo, hi) are not the stream's:
            // the granule maxima read them as zeros (a zero is never a strict maximum and
            // never beats one; the byte-level tests below only read inside [lo, hi)).  The
            // buffer itself is never written by a thread: only the bulk copy writes it.
            const uint32_t vend = off0 + (uint32_t)(hi - lo);
            const uint32_t NG = nbytes / 16;
            // buffer offset of stream position x: x - lo + off0
            const int64_t cbase = (int64_t)off0 - (int64_t)lo;
            const uint32_t c_lo = (uint32_t)((int64_t)ca + cbase), c_hi = (uint32_t)((int64_t)cb + cbase);
            if (h >= 31) {
                const uint32_t K0 = (uint32_t)((h - 15) / 16);  // granules wholly inside each window
                // blocks of MX_BG granules: for every granule j of block b, the blocks
                // b - NBK .. b + NBK lie wholly inside the granules [j - K0, j + K0]
                const uint32_t NBK = K0 >= MX_BG - 1 ? (K0 - (MX_BG - 1)) / MX_BG : 0;
                const uint32_t NB = (NG + MX_BG - 1) / MX_BG;
                // 1. granule maxima (the Extreme Byte Search leaf, DPX byte maxima), and the
                //    block maxima from the MX_BG lanes of a block (consecutive granules)
                for (uint32_t j0 = 0; j0 < NG; j0 += MX_THREADS) {  // uniform trip count (shuffles)
                    const uint32_t j = j0 + tid;
                    uint32_t m = 0;
                    if (j < NG) {
                        uint4 v = *reinterpret_cast<const uint4 *>(buf + 16 * j);
                        if (j == 0 || j == NG - 1) {  // keep bytes [off0, vend) of the granule
                            uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const uint32_t x = 16 * j + k;
                                if (x < off0 || x >= vend) w[k >> 2] &= ~(0xFFu << (8 * (k & 3)));
                            }
                            v = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                        m = vext16<true>(v);
                        gm[j] = (uint8_t)m;
                    }
#pragma unroll
                    for (int o = 1; o < MX_BG; o <<= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
                    if ((tid & (MX_BG - 1)) == 0 && j < NG) bm[j / MX_BG] = (uint8_t)m;
                }
                __syncthreads();
                // 2. block filter: a local maximum of block b is the block's maximum (the block
                //    lies inside its windows) and beats blocks b-NBK..b+NBK; survivors are listed
                //    (windows shorter than a block, K0 < MX_BG - 1: granule by granule instead,
                //    a granule's maximum beating the K0 granules on each side; such granules
                //    are more than K0 apart, at most NG / 2 + 1 of them)
                const bool gmode = K0 < MX_BG - 1;
                if (gmode) {
                    for (uint32_t g = c_lo / 16 + tid; g < (c_hi + 15) / 16; g += MX_THREADS) {
                        const uint32_t m = gm[g];
                        bool ok = m != 0u && g >= K0 && g + K0 < NG;
                        for (uint32_t k = 1; k <= K0 && ok; ++k) ok = gm[g - k] < m && gm[g + k] < m;
                        if (ok) surv[atomicAdd(&s_ns, 1u)] = (uint16_t)g;
                    }
                } else {
                    const uint32_t b_lo = (c_lo / 16) / MX_BG, b_hi = ((c_hi + 15) / 16 + MX_BG - 1) / MX_BG;
                    for (uint32_t b = b_lo + tid; b < b_hi; b += MX_THREADS) {
                        const uint32_t m = bm[b];
                        bool ok = m != 0u && b >= NBK && b + NBK < NB;
                        for (uint32_t k = 1; k <= NBK && ok; ++k) ok = bm[b - k] < m && bm[b + k] < m;
                        if (ok) surv[atomicAdd(&s_ns, 1u)] = (uint16_t)b;
                    }
                }
                __syncthreads();
                // 3. one warp per surviving block: the exact test of its maximum (PAPER.md l.196:
                //    greater than every byte of both h-byte windows), in any order; ranked below
                const uint32_t ns = s_ns;
                const int lane = tid & 31;
                for (uint32_t i = (uint32_t)tid >> 5; i < ns; i += MX_THREADS / 32) {
                    uint32_t j, m;
                    if (gmode) {
                        j = surv[i];
                        m = gm[j];
                    } else {
                        const uint32_t b = surv[i];
                        m = bm[b];
                        // the block's granule holding m (two of them: neither byte is a strict maximum)
                        const uint32_t jb = MX_BG * b + (uint32_t)lane;
                        const uint32_t hg = __ballot_sync(0xFFFFFFFFu, lane < MX_BG && jb < NG && gm[jb] == m);
                        if (__popc(hg) != 1) continue;
                        j = MX_BG * b + (uint32_t)(__ffs(hg) - 1);
                    }
                    if (j < K0 || j + K0 >= NG) continue;
                    // the granule's byte holding m, unique (its bytes are within 15 <= h)
                    const uint32_t hb = __ballot_sync(0xFFFFFFFFu, lane < 16 && buf[16 * j + lane] == m);
                    if (__popc(hb) != 1) continue;
                    const uint32_t tpos = 16 * j + (uint32_t)(__ffs(hb) - 1);
                    if (tpos < c_lo || tpos >= c_hi) continue;
                    // every other granule of [j-K0, j+K0], then the window bytes outside them
                    bool ok = true;
                    for (uint32_t q = j - K0 + (uint32_t)lane; q <= j + K0; q += 32) ok = ok && (q == j || gm[q] < m);
                    const uint32_t l0 = tpos - (uint32_t)h, l1 = 16 * (j - K0);
                    for (uint32_t x = l0 + (uint32_t)lane; x < l1; x += 32) ok = ok && buf[x] < m;
                    const uint32_t r0b = 16 * (j + K0 + 1), r1 = tpos + (uint32_t)h;
                    for (uint32_t x = r0b + (uint32_t)lane; x <= r1; x += 32) ok = ok && buf[x] < m;
                    if (__all_sync(0xFFFFFFFFu, ok) && lane == 0) {
                        const uint32_t k = atomicAdd(&s_cnt, 1u);
                        if (k < Q.ccap) cand[k] = (uint16_t)(tpos - c_lo + (uint32_t)(ca - a));
                    }
                }
                __syncthreads();
                count = s_cnt < Q.ccap ? s_cnt : Q.ccap;
                // rank by position (distinct), written straight into the tile's slot
                for (uint32_t i = tid; i < count; i += MX_THREADS) {
                    const uint16_t v = cand[i];
                    uint32_t r = 0;
                    for (uint32_t k = 0; k < count; ++k) r += cand[k] < v;
                    X.qt[t * Q.ccap + r] = v;
                }
                ranked = true;
            } else {
                // short windows: every position, exact test (early exit at the first byte not smaller)
                for (uint32_t r0 = c_lo; r0 < c_hi; r0 += MX_THREADS) {
                    const uint32_t x = r0 + tid;
                    bool ok = false;
                    if (x < c_hi) {
                        const uint32_t m = buf[x];
                        ok = m > 0;
                        for (uint32_t k = 1; k <= (uint32_t)h && ok; ++k) ok = buf[x - k] < m && buf[x + k] < m;
                    }
                    uint32_t tot;
                    const uint32_t o = mx_block_scan(ok ? 1u : 0u, tot, s_scr);
                    if (ok && count + o < Q.ccap) cand[count + o] = (uint16_t)(x - c_lo + (uint32_t)(ca - a));
                    count += tot;
                }
            }
        }
        __syncthreads();  // the last round's candidates are written
        // this tile's maxima into its own slot (k_maxp_gather orders the slots)
        if (!ranked)
            for (uint32_t i = tid; i < count; i += MX_THREADS) X.qt[t * Q.ccap + i] = cand[i];
        if (tid == 0) X.qn[t] = count;
        __syncthreads();
    }
    if (tid == 0) mbar_inval(&bar);
}

// K1b: the elements, file by file: one thread per scan tile, a block scan of
// the tile counts and a decoupled look-back over the CTAs give the tile's
// first element; file F's start element sits before its first tile's maxima.
__global__ void __launch_bounds__(MX_GTILES) k_maxp_gather(MaxpGeo Q, MaxpWork X) {
    __shared__ uint32_t s_tile, s_scr[64];
    __shared__ uint64_t s_slot;
    if (threadIdx.x == 0) s_tile = atomicAdd(X.ctrl + 3, 1u) + 1u;  // CTAs in ticket order
    __syncthreads();
    const uint64_t ntot = X.tfirst[Q.nfiles];
    const uint64_t g = s_tile;
    const uint64_t t = g * MX_GTILES + threadIdx.x;
    const uint32_t n = t < ntot ? X.qn[t] : 0u;
    uint32_t tot;
    const uint32_t o = mx_block_scan(n, tot, s_scr);
    const uint64_t excl = mx_tile_prefix(X.tst, g, tot, &s_slot);
    if (t < ntot) {
        const uint32_t F = Q.file_off != nullptr ? X.tfile[t] : 0u;
        const uint64_t t0 = Q.file_off != nullptr ? X.tfirst[F] : 0u;
        const uint64_t e0 = excl + o + F + 1;  // maxima before this tile, plus the starts of files 0..F
        if (t == t0) {                          // the file's start element
            X.qx[e0 - 1] = -1;
            X.efile[e0 - 1] = F;
            X.estart[F] = e0 - 1;
        }
        const int64_t a = (int64_t)(t - t0) * MX_TILE;
        for (uint32_t i = 0; i < n; ++i) {
            X.qx[e0 + i] = a + X.qt[t * Q.ccap + i];
            X.efile[e0 + i] = F;
        }
    }
    if ((g + 1) * MX_GTILES >= ntot && threadIdx.x == 0) {
        *X.nq = excl + tot + Q.nfiles;
        X.estart[Q.nfiles] = excl + tot + Q.nfiles;
    }
}

// Where the chunk run that starts at element e ends: its start s is the file
// start (qx[e] < 0) or right after the maximum qx[e]; the first maximum q[j] in
// [s+h, s+M) ends the chunk; capped chunks move s by M; maxima within h of a
// start are skipped (M3).  f = jend (the next file's start element): the run
// ends at the file end.  Mirrors the chain rule of PAPER.md §2.1.2 l.196 with
// R5's cap, one start at a time.
__device__ __forceinline__ void maxp_run(const MaxpGeo &Q, const int64_t *q, uint64_t L, uint64_t e, uint64_t jend,
                                         int64_t &f, uint64_t &ncap) {
    const uint64_t h = Q.h, M = Q.M;
    uint64_t s = q[e] < 0 ? 0 : (uint64_t)q[e] + 1;
    uint64_t j = e + 1;
    ncap = 0;
    for (;;) {
        while (j < jend && (uint64_t)q[j] < s + h) ++j;      // too close to the chunk start
        const uint64_t limit = (L - s < M) ? L : s + M;
        if (j < jend && (uint64_t)q[j] < limit) {            // content boundary right after q[j]
            f = (int64_t)j;
            return;
        }
        if (limit == L) {                                    // the chunk ends at the file end
            f = (int64_t)jend;
            return;
        }
        if (j >= jend) {                                     // capped chunks up to the file end
            ncap += (L - s - 1) / M;
            f = (int64_t)jend;
            return;
        }
        const uint64_t k = ((uint64_t)q[j] - s) / M;         // >= 1: capped chunks before q[j]'s
        ncap += k;
        s += k * M;
    }
}

// K2: every element's run; the runs that skip a maximum, listed in order.
__global__ void __launch_bounds__(MX_ETILE) k_maxp_link(MaxpGeo Q, MaxpWork X) {
    __shared__ uint32_t s_tile, s_scr[64];
    __shared__ uint64_t s_slot;
    const uint64_t nE = *X.nq;
    const uint64_t ntl = (nE + MX_ETILE - 1) / MX_ETILE;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(X.ctrl + 1, 1u) + 1u;
        __syncthreads();
        const uint64_t t = s_tile;
        if (t >= ntl) break;
        const uint64_t e = t * MX_ETILE + threadIdx.x;
        bool jump = false;
        if (e < nE) {
            const uint32_t F = X.efile[e];
            uint64_t off, L;
            mx_file(Q, F, off, L);
            int64_t f;
            uint64_t nc;
            maxp_run(Q, X.qx, L, e, X.estart[F + 1], f, nc);
            X.f[e] = f;
            X.ncap[e] = nc;
            jump = f > (int64_t)e + 1;
        }
        uint32_t tot;
        const uint32_t o = mx_block_scan(jump ? 1u : 0u, tot, s_scr);
        const uint64_t excl = mx_tile_prefix(X.lst, t, tot, &s_slot);
        if (jump) X.jl[excl + o] = (int64_t)e;
        if (t == ntl - 1 && threadIdx.x == 0) *X.nj = excl + tot;
        __syncthreads();
    }
}

// K3 (one CTA): the skipping runs in stream order.  A run is on the chain
// unless an earlier run on the chain jumped over its element; the elements a
// chain run jumps over are marked off the chain.  (Runs skip maxima only in
// capped stretches, so the list is short; a run never passes its file's end.)
constexpr int MX_PATH_BATCH = 2048;  // skipping runs staged in shared memory per round
__global__ void __launch_bounds__(256) k_maxp_path(MaxpGeo Q, MaxpWork X) {
    __shared__ int64_t s_i[MX_PATH_BATCH], s_f[MX_PATH_BATCH];
    __shared__ int64_t s_cur;
    const uint64_t nj = *X.nj;
    if (threadIdx.x == 0) s_cur = INT64_MIN;  // f of the last run on the chain that skipped maxima
    for (uint64_t k0 = 0; k0 < nj; k0 += MX_PATH_BATCH) {
        const uint64_t m = nj - k0 < MX_PATH_BATCH ? nj - k0 : MX_PATH_BATCH;
        __syncthreads();
        for (uint64_t k = threadIdx.x; k < m; k += blockDim.x) {
            const int64_t e = X.jl[k0 + k];
            s_i[k] = e;
            s_f[k] = X.f[e];
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            int64_t cur = s_cur;
            for (uint64_t k = 0; k < m; ++k) {
                const int64_t e = s_i[k];
                if (e < cur) continue;  // inside that run: not on the chain
                const int64_t f = s_f[k];
                for (int64_t x = e + 1 + (int64_t)threadIdx.x; x < f; x += 32) X.on[x] = 0;
                cur = f;
            }
            if (threadIdx.x == 0) s_cur = cur;
        }
    }
}

// K4: boundaries.  Element e on the chain contributes its capped chunks and the
// chunk that ends its run (a file start of an empty file: none); a decoupled
// look-back over the counts gives the output offsets (a batch: a file's start
// element's offset is the file's first output); each warp writes its 32
// elements' runs with all lanes.  Ends are file-relative.
__global__ void __launch_bounds__(MX_ETILE) k_maxp_write(MaxpGeo Q, MaxpWork X, uint64_t *bounds, uint64_t cap,
                                                         uint64_t *d_count) {
    __shared__ uint32_t s_tile, s_scr[64];
    __shared__ uint64_t s_slot;
    const uint64_t nE = *X.nq;
    const uint64_t ntl = (nE + MX_ETILE - 1) / MX_ETILE;
    const int lane = threadIdx.x & 31;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(X.ctrl + 2, 1u) + 1u;
        __syncthreads();
        const uint64_t t = s_tile;
        if (t >= ntl) break;
        const uint64_t e = t * MX_ETILE + threadIdx.x;
        uint64_t n = 0, nc = 0, s = 0, end = 0;
        bool fstart = false;
        uint32_t F = 0;
        if (e < nE) {
            F = X.efile[e];
            const int64_t qe = X.qx[e];
            fstart = qe < 0;
            uint64_t off, L;
            mx_file(Q, F, off, L);
            if (X.on[e] != 0 && L > 0) {
                nc = X.ncap[e];
                n = nc + 1;
                s = fstart ? 0 : (uint64_t)qe + 1;
                const int64_t f = X.f[e];
                end = f < (int64_t)X.estart[F + 1] ? (uint64_t)X.qx[f] + 1 : L;
            }
        }
        // per-thread counts can exceed 32 bits only for runs of > 4 G capped chunks
        uint32_t tot;
        const uint32_t o32 = mx_block_scan((uint32_t)n, tot, s_scr);
        const uint64_t excl = mx_tile_prefix(X.wst, t, tot, &s_slot);
        const uint64_t o = excl + o32;
        if (fstart && X.bo) X.bo[F] = o;
        for (int r = 0; r < 32; ++r) {
            const uint64_t rn = __shfl_sync(0xFFFFFFFFu, n, r);
            if (rn == 0) continue;
            const uint64_t ro = __shfl_sync(0xFFFFFFFFu, o, r), rs = __shfl_sync(0xFFFFFFFFu, s, r);
            const uint64_t rc = rn - 1, re = __shfl_sync(0xFFFFFFFFu, end, r);
            for (uint64_t k = lane; k <= rc; k += 32) {
                const uint64_t idx = ro + k;
                if (idx < cap) bounds[idx] = k < rc ? rs + (k + 1) * Q.M : re;
            }
        }
        if (t == ntl - 1 && threadIdx.x == 0) {
            *d_count = excl + tot;
            if (X.bo) X.bo[Q.nfiles] = excl + tot;
        }
        __syncthreads();
    }
}
