// cdc_kphase.cuh -- K-phase speculation: a single stream with a long window
// (included by cdc_kernels.cu; DESIGN.md §6 "K-phase speculation").
//
// On saturated bytes (uniform, or any stream where the window nearly always
// holds the saturating value) a chain started at an arbitrary offset meets the
// true chain only after ~(w / 362)^2 chunks: the phase difference of two
// chains random-walks over one chunk length (RAM §2.1.2 l.198: the chunk ends
// after the first 0xFF past the window; AE l.169: w bytes after the first
// 0xFF of [s, s+w]).  With one speculative chain per segment the halos then
// cost many segments' worth of walking, and the longest one sets the call's
// time.  Here every segment g starts K chains, at p_g + k D (D = (w + 256) / K,
// about a chunk length / K): the chain entering a segment lies between two of
// them, a gap of ~D instead of ~w, and meets one after ~K^2 fewer chunks.
//
// Nodes.  Chain (g, k) is node v = g K + k.  Its walker (k_kspec: one warp per
// node, taken in ticket order) records the chain's starts in list(v) (offsets
// from p_g; the body [start, p_{g+1}) and then the halo), and stops when
//   * a start lies on the chain of sibling (g, k+1) (body; a sibling that
//     stopped forwards to the one it met).  Chain k+1 started D bytes further
//     on and its walker first (tickets take a segment's nodes from k = K-1
//     down), so its entries at our positions are normally written already:
//     the trailing chain of two that merged sees it within a chunk.  The chain
//     K-1 of the segment probes nothing in its body; or
//   * a start past p_{g+1} lies on the chain of one of segment j's K nodes
//     (j = the segment holding it; halo), or
//   * the stream ends (KN_END), or the halo exceeds its cap (KN_UNSYNC).
// It publishes nxt(v) (the node met, or KN_*), idx(v) (the index of the
// meeting start in list(nxt(v))) and then pub(v) = its entry count (release).
// From a common start on two chains are identical, so the true chain is a
// path of pieces: from node 0 at index 0, list(v)[i .. cnt(v)), then node
// nxt(v) from idx(v), ... until a node with KN_END.
//
// Resolution (all on the device, no host round trip):
//   k_kres1  one warp per block of KB segments: for every node of the block,
//            the first node its path reaches outside the block and the sum of
//            val(u) = cnt(u) - idx(u) over the path's nodes inside the block;
//   k_kres2  one CTA: follows node 0's path block by block (level-1 records in
//            shared memory) and writes each visited block's entry (node,
//            index, output offset) and the boundary count; a KN_UNSYNC node on
//            the path opens the gate of the ordinary pipeline (launched behind,
//            it does all the work again and writes the output);
//   k_kres3  one warp per block: from its entry, writes the true chain's
//            starts inside the block as chunk end offsets.
#pragma once
// (included inside namespace cdc)

constexpr uint32_t KN_VOID = 0xFFFFFFFDu;   // a node whose start lies past its segment (never reached)
constexpr uint32_t KN_UNSYNC = 0xFFFFFFFEu; // the halo gave up (cap) or the list filled up
constexpr uint32_t KN_END = 0xFFFFFFFFu;    // the chain reached the stream's end
constexpr uint32_t KPUB_OPEN = 0xFFFFFFFFu;
constexpr int KB = 32;                      // segments per resolution block
constexpr int KRES1_WARPS = 8;
constexpr int KP_MAXK = 8;
constexpr uint32_t KNODE_MAX = 24576;       // k_kres2 keeps 8 bytes per node in shared memory
// level-1 records pack the exit node and index into 16 bits each
constexpr uint32_t KX_VOID = 0xFFFDu, KX_UNSYNC = 0xFFFEu, KX_END = 0xFFFFu;

struct KGeo {
    const uint8_t *data;
    uint64_t L;         // stream length
    uint32_t G, K, D;   // segments, chains per segment, start spacing
    uint32_t capk;      // list capacity per node (a multiple of 4)
    uint32_t w;
    uint64_t max_size;
    uint64_t Hk;        // halo cap (bytes past the segment end)
    int sparse;
    const uint32_t *skip;  // non-null: the dense-index mode's gate; 0 there = the output is written already
};
// (read before griddepcontrol.wait: the gate is final before any kernel behind k_dense_finish can start,
// see Geometry::gate0 in cdc_kernels.cu)
__device__ __forceinline__ bool kskip(const KGeo &Q) { return Q.skip != nullptr && __ldcg(Q.skip) == 0u; }
struct KWork {
    uint32_t *list;     // N x capk: starts - p_g (reset to LIST_EMPTY)
    uint32_t *pub;      // N: KPUB_OPEN, then the node's entry count (reset)
    uint32_t *ctrl;     // [0] node ticket (reset to ~0)
    uint32_t *nxt, *idx;// N: the node met and the index of the meeting start in its list
    uint32_t *bxi;      // N: level-1 exit (node16 << 16 | index16)
    int32_t *bval;      // N: level-1 sum of cnt - idx
    uint64_t *ent;      // NB x 2: entry (node | index << 32, ~0 = none) and output offset
    uint32_t *gate;     // 1 = the ordinary pipeline must run (written by k_kres2)
};

__device__ __forceinline__ int64_t kseg_start(const KGeo &Q, uint64_t g) { return seg_start(g, Q.G, Q.L); }
// segment holding stream position e
__device__ __forceinline__ uint32_t kseg_of(const KGeo &Q, int64_t e) {
    int64_t k = e / (int64_t)(Q.L / Q.G);
    if (k > (int64_t)Q.G - 1) k = (int64_t)Q.G - 1;
    while (k > 0 && kseg_start(Q, (uint64_t)k) > e) --k;
    while (k + 1 < (int64_t)Q.G && kseg_start(Q, (uint64_t)k + 1) <= e) ++k;
    return (uint32_t)k;
}

__device__ __forceinline__ uint4 ld_relaxed_v4(const uint32_t *p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

// Body probe of node (g, k): is relative start r on the chain of sibling
// (g, k+1)?  Warp-cooperative scan of the sibling's list from a monotone
// cursor (32 entries per window, one per lane).  When the sibling stopped
// because it met another sibling of the segment, the probe moves on to that
// one from the meeting index (its list holds the rest of the chain).
// Returns 1 (node, index set), 0 (not on it), -1 (not decidable yet).
struct KSib {
    uint32_t t;       // node probed (KN_END: none left)
    uint32_t cursor;  // entries before it are < every r still to come
    uint32_t wb, wv;  // cached window: lane holds entry wb + lane (wb = ~0: none)

    __device__ int probe(const KGeo &Q, const KWork &KW, uint32_t r, uint32_t &node, uint32_t &ix) {
        const int lane = lane_id();
        while (t != KN_END) {
            const uint32_t *lst = KW.list + (uint64_t)t * Q.capk;
            bool reloaded = false;  // the cached window was read again for this probe
            for (;;) {
                if (cursor >= Q.capk) break;
                const uint32_t B = cursor & ~31u;
                const bool mine = B + (uint32_t)lane < Q.capk;
                if (B != wb) {
                    wb = B;
                    wv = mine ? ld_relaxed_u32(lst + B + lane) : LIST_EMPTY;
                    reloaded = true;
                }
                const int off = (int)(cursor - B);
                const bool inwin = lane >= off;
                const bool valid = !inwin || wv != LIST_EMPTY;
                const uint32_t vm = __ballot_sync(0xFFFFFFFFu, valid);
                const uint32_t gm = __ballot_sync(0xFFFFFFFFu, inwin && valid && wv >= r);
                const int fi = vm == 0xFFFFFFFFu ? 32 : __ffs(~vm) - 1;
                const int fg = gm ? __ffs(gm) - 1 : 32;
                if (fg < fi) {
                    cursor = B + (uint32_t)fg;
                    if (__shfl_sync(0xFFFFFFFFu, wv, fg) == r) {
                        node = t;
                        ix = cursor;
                        return 1;
                    }
                    return 0;
                }
                if (fi < 32) {  // an entry not written (as cached) before any >= r
                    cursor = B + (uint32_t)fi;
                    if (!reloaded) {  // read the window again once: it may have been written since
                        wv = mine ? ld_relaxed_u32(lst + B + lane) : LIST_EMPTY;
                        reloaded = true;
                        continue;
                    }
                    break;
                }
                cursor = B + 32;
            }
            // the entry at the cursor is not written: still walking, or stopped before r
            const uint32_t pb = ld_acquire_u32(KW.pub + t);
            if (pb == KPUB_OPEN || cursor < pb) return -1;
            const uint32_t nx = KW.nxt[t];  // (visible: published before pub)
            if (nx < KN_VOID && nx / Q.K == t / Q.K) {  // it met a higher sibling: continue there
                cursor = KW.idx[t];
                t = nx;
                wb = ~0u;
                continue;
            }
            t = KN_END;  // it left the segment or ended: nothing more to meet here
        }
        return 0;
    }
};

// Halo probe: is stream position e a start of one of the K chains of the
// segment j holding it?  Lane m < K scans list(j K + m) from its own monotone
// cursor with a cached aligned group of four entries.
struct KSegProbe {
    int64_t lo, hi;   // segment j's range [p_j, p_{j+1}) (lo > hi: none yet)
    uint32_t j;
    uint32_t cm, cb;  // per lane: cursor, cached group (~0: none)
    uint4 cv;

    __device__ int probe(const KGeo &Q, const KWork &KW, int64_t e, uint32_t &node, uint32_t &ix) {
        const int lane = lane_id();
        if (e < lo || e >= hi) {
            j = kseg_of(Q, e);
            lo = kseg_start(Q, j);
            hi = kseg_start(Q, (uint64_t)j + 1);
            cm = 0;
            cb = ~0u;
        }
        const uint32_t r = (uint32_t)(e - lo);
        int res = 0;
        if ((uint32_t)lane < Q.K) {
            const uint32_t u = j * Q.K + (uint32_t)lane;
            const uint32_t *lst = KW.list + (uint64_t)u * Q.capk;
            for (;;) {
                if (cm >= Q.capk) break;
                if (cb != (cm & ~3u)) {
                    cb = cm & ~3u;
                    cv = ld_relaxed_v4(lst + cb);
                }
                const uint32_t q = cm - cb;
                const uint32_t x = q == 0 ? cv.x : q == 1 ? cv.y : q == 2 ? cv.z : cv.w;
                if (x == LIST_EMPTY) {
                    const uint32_t pb = ld_relaxed_u32(KW.pub + u);
                    cb = ~0u;  // read the group again next time
                    res = (pb != KPUB_OPEN && cm >= pb) ? 0 : -1;
                    break;
                }
                if (x < r) {
                    ++cm;
                    continue;
                }
                res = x == r ? 1 : 0;
                break;
            }
        }
        const uint32_t hit = __ballot_sync(0xFFFFFFFFu, res == 1);
        if (hit) {
            const int L = __ffs(hit) - 1;
            node = j * Q.K + (uint32_t)L;
            ix = __shfl_sync(0xFFFFFFFFu, cm, L);
            return 1;
        }
        return __any_sync(0xFFFFFFFFu, res < 0) ? -1 : 0;
    }
};

struct KEmit {
    const KGeo *Q;
    const KWork *KW;
    uint32_t k;
    int64_t p, pe;      // the node's segment [p, pe)
    uint32_t *lst;
    uint32_t cnt;
    uint32_t nx, nix;   // exit: node met (or KN_*) and the index of the meeting start
    KSib sib;
    KSegProbe seg;

    __device__ bool boundary(int64_t e) {
        uint32_t node = 0, ix = 0;
        if (e < pe) {
            if (k + 1 < Q->K && sib.probe(*Q, *KW, (uint32_t)(e - p), node, ix) == 1) {
                nx = node;
                nix = ix;
                return true;
            }
        } else {
            if ((uint64_t)(e - pe) >= Q->Hk) {
                nx = KN_UNSYNC;
                return true;
            }
            if (seg.probe(*Q, *KW, e, node, ix) == 1) {
                nx = node;
                nix = ix;
                return true;
            }
        }
        if (cnt >= Q->capk) {
            nx = KN_UNSYNC;
            return true;
        }
        if (lane_id() == 0) __stcg(lst + cnt, (uint32_t)(e - p));  // L2 store; readers use ld.relaxed.gpu
        ++cnt;
        return false;
    }
    __device__ bool in_halo() const { return false; }
    __device__ void end() { nx = KN_END; }
    __device__ void exhausted(int64_t) { nx = KN_UNSYNC; }
};

template <int ALGO>
__device__ void knode_walk(const KGeo &Q, const KWork &KW, const WarpRing &R, uint32_t v) {
    const int lane = lane_id();
    const uint32_t g = v / Q.K, k = v % Q.K;
    const int64_t p = kseg_start(Q, g), pe = kseg_start(Q, (uint64_t)g + 1);
    const int64_t s = p + (int64_t)k * Q.D;
    KEmit em;
    em.Q = &Q;
    em.KW = &KW;
    em.k = k;
    em.p = p;
    em.pe = pe;
    em.lst = KW.list + (uint64_t)v * Q.capk;
    em.cnt = 0;
    em.nx = KN_UNSYNC;
    em.nix = 0;
    em.sib.t = v + 1;
    em.sib.cursor = 0;
    em.sib.wb = ~0u;
    em.sib.wv = LIST_EMPTY;
    em.seg.lo = 1;
    em.seg.hi = 0;
    em.seg.j = 0;
    em.seg.cm = 0;
    em.seg.cb = ~0u;
    bool walk = true;
    if (s >= pe) {  // the segment is shorter than this start
        em.nx = KN_VOID;
        walk = false;
    } else {
        uint32_t node = 0, ix = 0;
        if (k + 1 < Q.K && em.sib.probe(Q, KW, (uint32_t)(s - p), node, ix) == 1) {  // the start itself
            em.nx = node;
            em.nix = ix;
            walk = false;
        } else {
            if (lane == 0) __stcg(em.lst, (uint32_t)(s - p));
            em.cnt = 1;
        }
    }
    unsigned long long *tm = g_timing ? g_timing + TM_STAMPS + (uint64_t)TM_PER_SEG * v : nullptr;
    if (tm && lane == 0) tm[0] = globaltimer();
    if (walk) {
        int64_t read_end = pe + (int64_t)Q.Hk + (int64_t)Q.max_size;
        if (g + 1 == Q.G || read_end > (int64_t)Q.L) read_end = (int64_t)Q.L;
        walk_chain<ALGO, STAGE, 2>(Q.sparse != 0, R, Q.data, (int64_t)Q.L, s, read_end, Q.w, Q.max_size, stream_policy(), em);
    }
    __syncwarp();
    if (lane == 0) {
        KW.nxt[v] = em.nx;
        KW.idx[v] = em.nix;
        st_release_u32(KW.pub + v, em.cnt);
        if (tm) {
            tm[1] = globaltimer();
            tm[2] = smid() | ((unsigned long long)em.cnt << 32);
        }
    }
    __syncwarp();
}

// K1 of the K-phase pipeline: warps take nodes from a ticket, segment-major,
// each segment's from k = K-1 down (a node's higher sibling, which it probes,
// was taken before it).
template <int ALGO>
__global__ void __launch_bounds__(SPEC_WARPS * 32, 1) k_kspec(KGeo Q, KWork KW) {
    extern __shared__ __align__(128) uint8_t smem[];
    if (threadIdx.x == 0) stamp(TM_SPEC_BEGIN);
    if (kskip(Q)) return;
    pdl_wait();  // the reset of the lists has completed
    if (threadIdx.x == 0) stamp(TM_SPEC_WAITED);
    const int warp = threadIdx.x >> 5, lane = lane_id();
    uint8_t *wbase = align_smem(smem) + warp * RING_SMEM;
    const WarpRing R{wbase, reinterpret_cast<uint64_t *>(wbase + RING_BYTES)};
    const uint32_t N = Q.G * Q.K;
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(KW.ctrl, 1u) + 1u;  // the counter starts at ~0
        t = __shfl_sync(0xFFFFFFFFu, t, 0);
        if (t >= N) break;
        knode_walk<ALGO>(Q, KW, R, t - t % Q.K + (Q.K - 1 - t % Q.K));  // a segment's nodes from k = K-1 down
    }
    pdl_trigger();
    if (lane == 0) stamp(TM_SPEC_END);
}

// Level 1: per block of KB segments, every node's first exit from the block
// (warp slot `ws` of KRES1_WARPS works on block b).
__device__ __forceinline__ void kres1_block(const KGeo &Q, const KWork &KW, int ws, uint32_t b,
                                            uint32_t (*s_nx)[KB * KP_MAXK], uint32_t (*s_ix)[KB * KP_MAXK],
                                            uint32_t (*s_cn)[KB * KP_MAXK]) {
    const int lane = lane_id();
    const uint32_t N = Q.G * Q.K;
    const uint32_t v0 = b * KB * Q.K, v1 = min(N, v0 + KB * Q.K);
    for (uint32_t v = v0 + lane; v < v1; v += 32) {
        s_nx[ws][v - v0] = KW.nxt[v];
        s_ix[ws][v - v0] = KW.idx[v];
        s_cn[ws][v - v0] = KW.pub[v];
    }
    __syncwarp();
    for (uint32_t v = v0 + lane; v < v1; v += 32) {
        uint32_t u = v, tx, ti;
        int32_t acc = 0;
        for (;;) {
            const uint32_t nx = s_nx[ws][u - v0];
            const uint32_t cn = s_cn[ws][u - v0];
            if (nx >= KN_VOID) {  // terminal
                acc += (int32_t)cn;
                tx = nx == KN_END ? KX_END : nx == KN_VOID ? KX_VOID : KX_UNSYNC;
                ti = 0;
                break;
            }
            const uint32_t ix = s_ix[ws][u - v0];
            acc += (int32_t)cn - (int32_t)ix;
            if (nx < v0 || nx >= v1) {
                tx = nx;
                ti = ix;
                break;
            }
            u = nx;
        }
        KW.bxi[v] = (tx << 16) | (ti & 0xFFFFu);
        KW.bval[v] = acc;
    }
    if (lane == 0) KW.ent[2 * b] = ~0ull;
    __syncwarp();
}
__global__ void __launch_bounds__(KRES1_WARPS * 32) k_kres1(KGeo Q, KWork KW) {
    __shared__ uint32_t s_nx[KRES1_WARPS][KB * KP_MAXK], s_ix[KRES1_WARPS][KB * KP_MAXK],
        s_cn[KRES1_WARPS][KB * KP_MAXK];
    if (kskip(Q)) return;
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5;
    const uint32_t NB = (Q.G + KB - 1) / KB;
    const uint32_t b = blockIdx.x * KRES1_WARPS + (uint32_t)warp;
    if (b >= NB) return;
    kres1_block(Q, KW, warp, b, s_nx, s_ix, s_cn);
}

// Level 2: node 0's path, block by block (one CTA; s_bxi / s_val: N words each).
__device__ __forceinline__ void kres2_path(const KGeo &Q, const KWork &KW, uint64_t *d_count, uint32_t *s_bxi,
                                           int32_t *s_val) {
    const uint32_t N = Q.G * Q.K;
    for (uint32_t v = threadIdx.x; v < N; v += blockDim.x) {
        s_bxi[v] = KW.bxi[v];
        s_val[v] = KW.bval[v];
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t v = 0, ix = 0;
    int64_t off = 0;
    uint32_t fail = 0;
    uint64_t total = 0;
    for (;;) {
        const uint32_t b = v / Q.K / KB;
        KW.ent[2 * b] = (uint64_t)v | ((uint64_t)ix << 32);
        KW.ent[2 * b + 1] = (uint64_t)off;
        const uint32_t bx = s_bxi[v];
        const uint32_t tx = bx >> 16, ti = bx & 0xFFFFu;
        const int64_t nxt_off = off + (int64_t)s_val[v] - (int64_t)ix + (int64_t)ti;
        if (tx == KX_END) {
            total = (uint64_t)(off + (int64_t)s_val[v] - (int64_t)ix);
            break;
        }
        if (tx >= KX_VOID) {  // KX_UNSYNC (KX_VOID is never met)
            fail = 1;
            break;
        }
        v = tx;
        ix = ti;
        off = nxt_off;
    }
    if (!fail) *d_count = total;
    *KW.gate = fail;
}
__global__ void __launch_bounds__(1024) k_kres2(KGeo Q, KWork KW, uint64_t *d_count) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t *s_bxi = reinterpret_cast<uint32_t *>(smem);
    if (kskip(Q)) return;  // (the ordinary pipeline behind looks at the dense gate first as well)
    pdl_wait();
    pdl_trigger();
    kres2_path(Q, KW, d_count, s_bxi, reinterpret_cast<int32_t *>(s_bxi + Q.G * Q.K));
}

// Level 3: one warp writes the true chain's starts inside block b.
__device__ __forceinline__ void kres3_block(const KGeo &Q, const KWork &KW, uint32_t b, uint64_t *bounds, uint64_t cap) {
    const int lane = lane_id();
    const uint64_t e0 = KW.ent[2 * b];
    if (e0 == ~0ull) return;  // the true chain jumps over this block
    uint32_t v = (uint32_t)e0, ix = (uint32_t)(e0 >> 32);
    uint64_t off = KW.ent[2 * b + 1];
    const uint32_t v0 = b * KB * Q.K, v1 = min(Q.G * Q.K, v0 + KB * Q.K);
    for (;;) {
        const uint32_t cn = KW.pub[v], nx = KW.nxt[v], nix = KW.idx[v];
        const uint64_t p = (uint64_t)kseg_start(Q, v / Q.K);
        const uint32_t *lst = KW.list + (uint64_t)v * Q.capk;
        for (uint32_t i = ix + (uint32_t)lane; i < cn; i += 32) {
            const uint64_t q = off + (i - ix);
            if (q >= 1 && q - 1 < cap) bounds[q - 1] = p + lst[i];
        }
        off += cn - ix;
        if (nx == KN_END) {  // the last chunk ends at the stream's end
            if (lane == 0 && off >= 1 && off - 1 < cap) bounds[off - 1] = Q.L;
            return;
        }
        if (nx >= KN_VOID || nx < v0 || nx >= v1) return;
        v = nx;
        ix = nix;
    }
}
__global__ void __launch_bounds__(256) k_kres3(KGeo Q, KWork KW, uint64_t *bounds, uint64_t cap) {
    if (kskip(Q)) return;
    pdl_wait();
    pdl_trigger();
    const uint32_t NB = (Q.G + KB - 1) / KB;
    const uint32_t b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= NB || *KW.gate != 0) return;
    kres3_block(Q, KW, b, bounds, cap);
}

// The three levels in one CTA, for streams of at most KRES_ALL_NB blocks (small
// streams, where three launches cost more than the work): level 1 by
// KRES1_WARPS warps over the blocks, level 2, level 3 by every warp; when a node
// on the true path gave up, the CTA resets the ordinary pipeline's lists
// ([rst, rst + n16)) instead, so that pipeline's own reset launch is not needed.
constexpr uint32_t KRES_ALL_NB = 32;
__global__ void __launch_bounds__(1024) k_kres_all(KGeo Q, KWork KW, uint64_t *d_count, uint64_t *bounds, uint64_t cap,
                                                   uint4 *rst, uint64_t n16) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t s_nx[KRES1_WARPS][KB * KP_MAXK], s_ix[KRES1_WARPS][KB * KP_MAXK],
        s_cn[KRES1_WARPS][KB * KP_MAXK];
    uint32_t *s_bxi = reinterpret_cast<uint32_t *>(smem);
    if (kskip(Q)) return;
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5;
    const uint32_t NB = (Q.G + KB - 1) / KB;
    if (warp < KRES1_WARPS)
        for (uint32_t b = (uint32_t)warp; b < NB; b += KRES1_WARPS) kres1_block(Q, KW, warp, b, s_nx, s_ix, s_cn);
    __syncthreads();  // (bxi, bval and the blocks' "no entry" marks, written and read by this CTA)
    kres2_path(Q, KW, d_count, s_bxi, reinterpret_cast<int32_t *>(s_bxi + Q.G * Q.K));
    __syncthreads();
    if (*KW.gate != 0) {
        const uint4 ones = make_uint4(~0u, ~0u, ~0u, ~0u);
        for (uint64_t i = threadIdx.x; i < n16; i += blockDim.x) rst[i] = ones;
        return;
    }
    for (uint32_t b = (uint32_t)warp; b < NB; b += blockDim.x >> 5) kres3_block(Q, KW, b, bounds, cap);
}
