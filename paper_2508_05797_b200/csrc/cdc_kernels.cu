// cdc_kernels.cu -- sm_100a kernels and the extern "C" ABI declared in include/cdc_b200.h.
//
// Pipeline of one cdc_chunk / cdc_chunk_batch call:
//   K0 k_seg_prefix  (batch only) segment table: nseg_f = ceil(L_f / S), prefix sums
//   K1 k_speculate   one warp per segment g: starts a chunk at the segment's first
//                    byte (speculation), walks the chain through the segment with a
//                    TMA-fed shared-memory ring, records the chain's starts (list(g)),
//                    publishes them (release) for the neighbour, then keeps walking
//                    past the segment end ("halo") until one of its starts is found
//                    in a later segment's published list (re-synchronisation: from a
//                    common start on, two chains are identical), the stream ends, or
//                    the halo exceeds its cap.
//   K2 k_fixup       exits at once when K1's fused look-back already wrote the output;
//                    otherwise its first CTA (resolve_block) re-checks undecided halos against the complete lists,
//                    runs fix-up walkers for halos that never met a later chain,
//                    resolves which segments the true chain passes through (from the
//                    stream start, following sync points), and scans the per-segment
//                    output counts.
//                    and then every CTA (write_segment, one warp per segment) writes its part of the true chain as
//                    exclusive chunk end offsets (uint64).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cdc_b200.h"
#include "cdc_device.cuh"

namespace cdc {

#ifndef CDC_SPEC_WARPS
#define CDC_SPEC_WARPS 16
#endif
constexpr int SPEC_WARPS = CDC_SPEC_WARPS;  // warps (segments) per CTA in k_speculate
#ifndef CDC_SPEC_CTAS_PER_SM
#define CDC_SPEC_CTAS_PER_SM 1
#endif
constexpr int SPEC_CTAS_PER_SM = CDC_SPEC_CTAS_PER_SM;  // resident k_speculate CTAs per SM (smem-bound)
// The batch kernel's walkers (mostly the sparse walk, whose chunks are bound by
// per-warp latency): 20 warps per SM with 2 x 5 KiB rings (96 registers)
// instead of 16 with 2 x 6 KiB (configs[3] 1.65 -> 1.54 ms; a single stream's
// ring walker is faster with the larger rings: configs[1] 0.0654 vs 0.0715 ms)
#ifndef CDC_BATCH_WARPS
#define CDC_BATCH_WARPS 20
#endif
#ifndef CDC_BATCH_STAGE
#define CDC_BATCH_STAGE 5120
#endif
constexpr int BATCH_WARPS = CDC_BATCH_WARPS;
constexpr int BATCH_STAGE = CDC_BATCH_STAGE;
static_assert(BATCH_WARPS * Ring<BATCH_STAGE>::SMEM + 128 <= 227 * 1024, "batch rings exceed shared memory");
static_assert(Ring<BATCH_STAGE>::BYTES >= SP_NSLOT * SP_SLOT && Ring<STAGE>::BYTES >= SP_NSLOT * SP_SLOT, "sparse-walk slots exceed a ring");
#ifndef CDC_HEAD_KEEP
#define CDC_HEAD_KEEP 12288
#endif
constexpr int HEAD_KEEP = CDC_HEAD_KEEP;  // bytes of each segment head kept in L2 for the halo re-read
constexpr int RESOLVE_THREADS = 1024;
#ifndef CDC_RING_OPAQUE
#define CDC_RING_OPAQUE 1  // keep k_speculate's ring pointer in a register (A/B knob)
#endif
#ifndef CDC_PUB_RELEASE
#define CDC_PUB_RELEASE 0  // 1: publish a list's final count with a release store (A/B)
#endif

// ------------------------------------------------------------------ workspace
struct Work {
    // per segment
    uint32_t *list;              // G x cap_list  starts relative to the segment start
    uint32_t *halo;              // G x cap_halo  starts relative to the segment end
    uint32_t *cnt, *hcnt;        // list / halo lengths
    unsigned long long *pub;     // PUB_OPEN, or the final list length
    unsigned long long *status;  // look-back words (ST_* flag | 62-bit signed value), reset to ~0
    uint32_t *ctrl;              // [0] CTA ticket counter, [1] fast path valid (~0) / failed (0); reset to ~0
    unsigned long long *fetched; // bytes k_speculate's walkers copied from global memory, minus one (reset to ~0)
    unsigned long long *grp;     // look-back group sums (reset to ~0)
    uint32_t *tblk;              // T-mode: per block of 32 segments, tables published (reset to ~0)
    int32_t *sj;                 // sync target segment, or SJ_* code
    uint32_t *sa, *sb;           // halo entries before the sync point; its index in list(sj)
    uint32_t *entry, *tail, *wcnt, *jump_entry;
    uint64_t *woff;              // walker entries offset into pool
    uint32_t *ocnt;              // serial fix-up walker entries (pool B) per segment
    uint64_t *ooff;              // their offset into pool B
    uint64_t *poolb;             // serial fix-up walker starts (file relative), sized for the whole stream
    uint8_t *skipped;
    uint64_t *seg_out;           // G+1 exclusive scan of output counts
    uint32_t *exc;               // compacted exceptional segments
    uint32_t *ranges;            // skip ranges (pairs)
    uint32_t *pool;              // fix-up walker starts: segment g's slice [g cap_halo, (g+1) cap_halo), relative to seg_end
    uint64_t *seg_first;         // nfiles+1 (batch)
    uint32_t *seg_file;          // G: file of each segment (batch)
    uint32_t *lpt;               // batch: long segments by size class (LptLists; counters in tnx, bitmap in tblk)
    uint64_t *lofs;              // G+1: first list entry of each segment (batch: lists sized by
                                 // segment length); null for a single stream (g * cap_list)
    uint64_t *file_out;          // nfiles+1 (single stream: internal)
    uint32_t *misc;              // [0] G, [1] n_exc, [2] n_ranges, [3] overflow flags
    // transfer tables (T-mode, saturated streams): per segment TK candidates
    uint32_t *tl;                // G x TK link: candidate k of g -> candidate of g+1 (T_END, T_BAD)
    uint32_t *tn;                // G x TK chain starts of candidate k inside the segment
    uint32_t *tk;                // G: table rows in use (candidates, then entries from the previous segment)
    int64_t *tex;                // G x TEX: exits of segment g that are not candidates of g+1 (its extra entries)
    uint32_t *tnx;               // G: their count, published after phase 1 (reset to ~0)
    uint32_t *tp, *tq;           // G x TK: for entry k of the segment's block, its entry candidate and
                                 // the chain starts in the block before it
    uint32_t *tbc, *tbs;         // NB x TK: block tables (entry -> next block's entry, starts inside)
    uint32_t *tbe;               // NB: the true chain's entry of each block (the scan)
    uint64_t *tbo;               // NB: its output index
    uint64_t cap_list, cap_halo, pool_cap, max_segs, exc_cap, poolb_cap;
};

enum : int32_t { SJ_UNSYNCED = -1, SJ_STREAM_END = -2, SJ_LAST = -3, SJ_TABLE = -4 };
constexpr int DYN_TICKET = 9;  // ctrl[9] (reset to ~0): a batch's per-warp segment tickets

// Largest-first order of a batch's long segments (k_speculate's tickets): a
// segment of at least 2^LPT_MIN_LOG2 bytes goes into the list of its size
// class b = min(floor(log2(len)) - LPT_MIN_LOG2, LPT_CLASSES - 1); tickets take
// the classes from the largest down, then the other segments in file order.
// A walker that starts a 16 MiB file last would otherwise finish alone, long
// after every other walker (the longest walks set the batch's tail).
constexpr int LPT_MIN_LOG2 = 20, LPT_CLASSES = 6;
__host__ __device__ __forceinline__ uint64_t lpt_cap(uint64_t total, int b) {
    return (total >> (LPT_MIN_LOG2 + b)) + 1;
}
__host__ __device__ __forceinline__ uint64_t lpt_base(uint64_t total, int b) {
    uint64_t o = 0;
    for (int i = 0; i < b; ++i) o += lpt_cap(total, i);
    return o;
}
struct LptLists {
    uint32_t *cnt;   // LPT_CLASSES counters (reset to ~0)
    uint32_t *map;   // one bit per segment, cleared for a listed one (reset to all ones)
    uint32_t *list;  // class b: [lpt_base(b), lpt_base(b) + lpt_cap(b))
    uint64_t total;  // batch bytes
};


// dynamic shared memory follows the kernel's static shared variables: round the
// ring up to 128 bytes (TMA destinations need 16, LDS.128 16; launches add 128)
__device__ __forceinline__ uint8_t *align_smem(uint8_t *p) {
    return reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(p) + 127) & ~static_cast<uintptr_t>(127));
}

struct Geometry {
    const uint8_t *data;
    const uint64_t *file_off;  // null => single stream of length L
    uint64_t L;
    uint64_t total;  // bytes of the stream or batch (as planned)
    uint64_t nfiles;
    uint64_t S;      // segment bytes
    uint64_t Hmax;   // halo cap
    uint32_t w;
    uint64_t max_size;
    int tmode;       // walkers may try transfer tables (single stream, one co-resident wave)
    int sparse;      // walkers start with the sparse walk (sparse_chain; long windows)
    const uint32_t *gate;  // non-null: run only if *gate != 0 (the fallback behind the K-phase pipeline)
    // non-null: the dense-index mode's gate, final before any kernel behind k_dense_finish can start (each
    // of them triggers its dependents only after it started, k_dense_finish only after its wait for the
    // resolver), so it is read before griddepcontrol.wait: behind a shut gate the chain of PDL launches
    // collapses instead of each kernel waiting for the one before it
    const uint32_t *gate0;
};
__device__ __forceinline__ bool gate0_shut(const uint32_t *g0) { return g0 != nullptr && __ldcg(g0) == 0u; }

__device__ __forceinline__ void file_bounds(const Geometry &G, uint64_t f, uint64_t &off, uint64_t &len) {
    if (G.file_off == nullptr) {
        off = 0;
        len = G.L;
    } else {
        off = G.file_off[f];
        len = G.file_off[f + 1] - off;
    }
}
// Segments of a file of `len` bytes: n = floor(len / S), at least one.  Segment
// k covers [start(k), start(k+1)) with start(k) = k floor(len / n) rounded down
// to 4 KiB (16 B for short files), the last one ending at len: lengths differ
// by less than one alignment unit plus n bytes (none is tiny, none twice as
// long) and every start is aligned for the TMA ring.
__host__ __device__ __forceinline__ uint64_t nseg_of(uint64_t len, uint64_t S) {
    return len == 0 ? 0 : (len < S ? 1 : len / S);
}
__host__ __device__ __forceinline__ int64_t seg_start(uint64_t k, uint64_t n, uint64_t len) {
    if (n == 1) return k >= 1 ? (int64_t)len : 0;  // (most batch files: no 64-bit division)
    const uint64_t q = len / n;
    const uint64_t align = q >= (64u << 10) ? 4095u : 15u;
    return k >= n ? (int64_t)len : (int64_t)((k * q) & ~align);
}

__device__ __forceinline__ void seg_first_of(const Geometry &G, const Work &W, uint64_t f, uint64_t &a,
                                             uint64_t &b) {
    if (G.file_off == nullptr) {
        a = 0;
        b = nseg_of(G.L, G.S);
    } else {
        a = W.seg_first[f];
        b = W.seg_first[f + 1];
    }
}
__device__ __forceinline__ uint64_t total_segs(const Geometry &G, const Work &W) {
    return G.file_off == nullptr ? nseg_of(G.L, G.S) : W.seg_first[G.nfiles];
}
// file containing segment g (batch: the map written by k_seg_prefix)
__device__ __forceinline__ uint64_t file_of_seg(const Geometry &G, const Work &W, uint64_t g) {
    if (G.file_off == nullptr) return 0;
    return W.seg_file[g];
}

struct SegInfo {
    uint64_t g, f, first, last;  // segment, file, file's first and last segment
    uint64_t foff, Lf;           // file offset in data and length
    int64_t p, seg_end;          // segment [p, seg_end) within the file
};
__device__ __forceinline__ SegInfo seg_info(const Geometry &G, const Work &W, uint64_t g) {
    SegInfo I;
    I.g = g;
    I.f = file_of_seg(G, W, g);
    uint64_t a, b;
    seg_first_of(G, W, I.f, a, b);
    I.first = a;
    I.last = b - 1;
    file_bounds(G, I.f, I.foff, I.Lf);
    I.p = seg_start(g - a, b - a, I.Lf);
    I.seg_end = seg_start(g - a + 1, b - a, I.Lf);
    return I;
}

// Published list of segment g: its first entry and its capacity.  A batch
// sizes each list by its segment's length (k_seg_prefix); a single stream's
// segments share one capacity.
__device__ __forceinline__ uint64_t list_off(const Work &W, uint64_t g) {
    return W.lofs ? W.lofs[g] : g * W.cap_list;
}
__device__ __forceinline__ uint64_t list_cap(const Work &W, uint64_t g) {
    return W.lofs ? W.lofs[g + 1] - W.lofs[g] : W.cap_list;
}

// global index and first byte (file-relative) of the segment of file position e
__device__ __forceinline__ int64_t seg_of_pos(const SegInfo &I, int64_t e, uint64_t, int64_t &pj) {
    const uint64_t n = I.last - I.first + 1;
    int64_t k = e / (int64_t)(I.Lf / n);
    if (k > (int64_t)n - 1) k = (int64_t)n - 1;
    while (k > 0 && seg_start(k, n, I.Lf) > e) --k;
    while (k + 1 < (int64_t)n && seg_start(k + 1, n, I.Lf) <= e) ++k;
    pj = seg_start(k, n, I.Lf);
    return (int64_t)I.first + k;
}

// Published lists.  list(g) holds the chunk starts of segment g's speculative
// chain that lie inside the segment (relative to its first byte, ascending);
// its entries are reset to LIST_EMPTY before every call (k_reset) and each
// is written once with a single 32-bit store, so a reader sees every entry
// either complete or empty.  pub(g) is PUB_OPEN until the walker has left its
// segment; then it holds the final entry count (st.release after the entries).
constexpr uint32_t LIST_EMPTY = 0xFFFFFFFFu;
constexpr unsigned long long PUB_OPEN = ~0ull;

// Re-synchronisation probe of a walker's chain against the published lists:
// warp-cooperative membership of boundary e in the list of the segment
// holding it, scanning from a monotone cursor (boundaries come in increasing
// order).  Returns 1 = found (idx set), 0 = not a member, -1 = undecidable yet
// (an entry the scan needs is not visible and the list is not known
// complete).  It caches the segment the last boundary fell in (its range, so
// no division while e stays inside it) and one aligned window of 32 entries
// of its list, one per lane (entries are written once, so a visible entry
// never changes; a window with an empty entry in use is read again).
struct ListProbe {
    int64_t j;           // segment of the last boundary (-1: none yet)
    int64_t lo, hi;      // its file-relative range [lo, hi)
    uint32_t cursor;     // monotone cursor in list(j)
    uint32_t wb;         // first entry index of the cached window (~0: none)
    uint32_t wv;         // this lane's cached entry wb + lane
    const uint32_t *lst; // list(j) and its capacity
    uint64_t cap;

    __device__ void reset() {
        j = -1;
        lo = hi = 0;
        cursor = 0;
        wb = ~0u;
    }
    __device__ int probe(const Work &W, const SegInfo &I, int64_t e, int64_t &jo, uint32_t &idx) {
        if (e < lo || e >= hi) {
            int64_t pj;
            j = seg_of_pos(I, e, 0, pj);
            lo = pj;
            const uint64_t n = I.last - I.first + 1;
            const uint64_t k = (uint64_t)(j - (int64_t)I.first);
            hi = k + 1 < n ? seg_start(k + 1, n, I.Lf) : (int64_t)I.Lf;
            cursor = 0;
            wb = ~0u;
            lst = W.list + list_off(W, (uint64_t)j);
            cap = list_cap(W, (uint64_t)j);
        }
        jo = j;
        const uint32_t r = (uint32_t)(e - lo);
        const int lane = lane_id();
        while (cursor < cap) {
            const uint32_t B = cursor & ~31u;
            const bool mine = (uint64_t)B + lane < cap;
            if (B != wb || __any_sync(0xFFFFFFFFu, mine && wv == LIST_EMPTY)) {
                wb = B;
                wv = mine ? ld_relaxed_u32(lst + B + lane) : LIST_EMPTY;
            }
            const int off = (int)(cursor - B);
            const bool inwin = lane >= off;
            const bool valid = !inwin || wv != LIST_EMPTY;  // entries before the cursor are < r
            const uint32_t vm = __ballot_sync(0xFFFFFFFFu, valid);
            const uint32_t gm = __ballot_sync(0xFFFFFFFFu, inwin && valid && wv >= r);
            const int fi = vm == 0xFFFFFFFFu ? 32 : __ffs(~vm) - 1;  // first empty entry
            const int fg = gm ? __ffs(gm) - 1 : 32;                  // first entry >= r
            if (fg < fi) {
                const uint32_t vL = __shfl_sync(0xFFFFFFFFu, wv, fg);
                cursor = B + (uint32_t)fg;
                if (vL == r) {
                    idx = cursor;
                    return 1;
                }
                return 0;
            }
            if (fi < 32) {
                const unsigned long long pw = ld_acquire_u64(W.pub + j);
                const uint32_t at = B + (uint32_t)fi;
                cursor = at;
                if (pw != PUB_OPEN && (uint64_t)pw <= at) return 0;  // the list ends before r
                return -1;
            }
            cursor = B + 32;
        }
        return 0;
    }
};

// ------------------------------------------------------------------ K1 emit policy
// Optional timing record (cdc_debug_timing): TM_STAMPS launch stamps
// (globaltimer; min slots preset to ~0 by the caller, max slots to 0), then
// TM_PER_SEG x u64 per segment {at start, at the end of the body walk (its
// first boundary at or past the segment end), at the end of the walk, at the
// end, smid | hcnt << 32, T-mode: index built, table built}.
__device__ unsigned long long *g_timing = nullptr;
constexpr int TM_STAMPS = 8;
constexpr int TM_PER_SEG = 7;
enum : int { TM_RESET_BEGIN, TM_RESET_END, TM_SPEC_BEGIN, TM_SPEC_WAITED, TM_SPEC_END, TM_FIX_BEGIN,
             TM_FIX_WAITED, TM_FIX_END };
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void stamp(int i) {  // one thread per CTA calls this
    unsigned long long *tm = g_timing;
    if (tm == nullptr) return;
    const unsigned long long t = globaltimer();
    if (i == TM_RESET_END || i == TM_SPEC_END || i == TM_FIX_END) atomicMax(tm + i, t);
    else atomicMin(tm + i, t);
}
struct SpecEmit {
    const Geometry *G;
    const Work *W;
    SegInfo I;
    uint32_t *list, *halo;
    unsigned long long *pub;
    uint32_t cnt, hcnt;
    int32_t sj;
    uint32_t sa, sb;
    ListProbe lp;
    bool published;
    unsigned long long *tbody;  // diagnostics: where to stamp the end of the body walk (or null)

    __device__ void publish() {
        if (!published) {
            if (lane_id() == 0) {
                // relaxed: a reader that sees the final count but not yet an
                // entry below it reads the entry as undecided and keeps walking
                // (ListProbe::probe returns -1), so no fence is needed
                if (CDC_PUB_RELEASE) st_release_u64(pub, (unsigned long long)cnt);
                else asm volatile("st.relaxed.gpu.u64 [%0], %1;" ::"l"(pub), "l"((unsigned long long)cnt) : "memory");
                if (tbody) *tbody = globaltimer();
            }
            published = true;
        }
    }
    __device__ bool boundary(int64_t e) {
        const int lane = lane_id();
        if (e < I.seg_end) {
            if (lane == 0) __stcg(list + cnt, (uint32_t)(e - I.p));  // L2 store; readers use ld.relaxed.gpu
            ++cnt;
            return false;
        }
        publish();
        const uint32_t h = (uint32_t)(e - I.seg_end);
        if (lane == 0) halo[hcnt] = h;
        ++hcnt;
        // re-synchronisation: is e a start of the chain of the segment holding it?
        int64_t j;
        uint32_t idx = 0;
        const int r = lp.probe(*W, I, e, j, idx);
        if (r == 1) {
            sj = (int32_t)j;
            sa = hcnt - 1;
            sb = idx;
            return true;
        }
        if ((uint64_t)h >= G->Hmax) {
            sj = SJ_UNSYNCED;
            return true;
        }
        return false;
    }
    __device__ bool in_halo() const { return published; }  // diagnostics (CDC_EVTIME)
    __device__ void end() { sj = (I.seg_end >= (int64_t)I.Lf) ? SJ_LAST : SJ_STREAM_END; }
    __device__ void exhausted(int64_t) { sj = SJ_UNSYNCED; }
};

__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}

// Programmatic dependent launch (PDL): the next kernel in the stream may be
// launched before this grid completes; it waits (griddepcontrol.wait) for the
// full completion and memory flush of its predecessor before touching its data.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// K0': reset of the published-list region (list entries, publish, look-back
// and ticket words) to all-ones; lets k_speculate launch early (PDL).
__global__ void __launch_bounds__(256) k_reset(uint4 *p, uint64_t n16, const uint32_t *gate,
                                               const uint32_t *gate0 = nullptr) {
    if (gate0 != nullptr && __ldcg(gate0) == 0u) return;  // (the dense-index mode wrote the output: see Geometry::gate0)
    if (gate) pdl_wait();  // (a gated reset is launched with PDL behind the kernels that write its gate)
    pdl_trigger();
    if (gate && *gate == 0) return;
    if (threadIdx.x == 0) stamp(TM_RESET_BEGIN);
    const uint4 ones = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = ones;
    if (threadIdx.x == 0) stamp(TM_RESET_END);
}

// Decoupled look-back words: the top two bits say what the low 62 bits (a
// signed value) hold.  k_reset leaves every word ~0 = not ready.
constexpr unsigned long long ST_AGG = 1ull << 62;   // a_g = (cnt + tail) - sb of this segment
constexpr unsigned long long ST_MASK = 3ull << 62;
__device__ __forceinline__ int64_t st_value(unsigned long long w) {
    return (int64_t)(w << 2) >> 2;  // sign-extend the 62-bit value
}
__device__ __forceinline__ unsigned long long st_word(unsigned long long flag, int64_t v) {
    return flag | ((unsigned long long)v & ~ST_MASK);
}
// a segment's status word: ST_AGG | sb << 32 | (uint32) a  (sb < 2^30, |a| < 2^31)
__device__ __forceinline__ unsigned long long seg_word(uint32_t sb, int64_t a) {
    return ST_AGG | ((unsigned long long)(sb & 0x3FFFFFFFu) << 32) | (unsigned long long)(uint32_t)(int32_t)a;
}
__device__ __forceinline__ int64_t seg_a(unsigned long long w) { return (int64_t)(int32_t)(uint32_t)w; }
__device__ __forceinline__ uint32_t seg_sb(unsigned long long w) { return (uint32_t)(w >> 32) & 0x3FFFFFFFu; }

// Output offset of segment g's first true chain start.  With entry(g) = sb(g-1)
// (the index in list(g) where segment g-1's chain met it; 0 at a file's first
// segment) and n(g) = cnt(g) + tail(g) - entry(g), the exclusive prefix sum of
// n telescopes to  sum_{h<g} a_h + sb(g-1)  with the purely local
// a_h = cnt(h) + tail(h) - sb(h).  Two-level scan: every segment publishes a_h
// (ST_AGG); the last segment of each group of 32 to finish publishes the
// group's sum (ST_AGG in grp).  A segment then waits for, and sums, the groups
// before its own and the members of its group before it: at most
// ceil(G/1024) + 1 independent loads per lane.  Returns sum_{h<g} a_h.
constexpr int LB_GROUP = 32;
#ifndef CDC_SLEEP0
#define CDC_SLEEP0 256
#endif
#ifndef CDC_SLEEPMAX
#define CDC_SLEEPMAX 1024
#endif
// look-back waits sleep (exponential backoff) instead of polling hard: waiting
// warps share their SM with walkers that are still running
constexpr uint32_t SLEEP0 = CDC_SLEEP0, SLEEPMAX = CDC_SLEEPMAX;
constexpr uint64_t LB_MAX_SEGS = 32768;  // beyond this k_fixup's resolver splices the chains

// all 32 lanes
// Group words: one 64-bit atomic accumulator per group of 32 segments holding
// (arrivals << 48) + sum of (a + LB_BIAS) over the arrived segments.  The
// reset leaves ~0, so the accumulated value is the word + 1.  A group is
// complete when its arrival count equals its size; its sum is then
// low48 - size * LB_BIAS.  (|a| < 2^24: a = cnt + tail - sb, each bounded by a
// segment's list or halo capacity.)
constexpr uint64_t LB_BIAS = 1ull << 24;
constexpr uint64_t LB_LOW48 = (1ull << 48) - 1;

// all 32 lanes
__device__ void publish_agg(Work &W, uint64_t g, uint64_t, int64_t a, uint32_t sb) {
    // Both words are self-contained (readers need nothing else these warps
    // wrote), so relaxed accesses suffice: no fences on the critical path.
    if (lane_id() == 0) {
        asm volatile("st.relaxed.gpu.u64 [%0], %1;" ::"l"(W.status + g), "l"(seg_word(sb, a)) : "memory");
        const unsigned long long add = (1ull << 48) + (unsigned long long)(a + (int64_t)LB_BIAS);
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(W.grp + g / LB_GROUP), "l"(add) : "memory");
    }
    __syncwarp();
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// All 32 lanes.  Relaxed loads issued together, then one acquire fence per
// lane.  Groups confirmed ready are not read again, and the wait backs off
// exponentially (a waiting warp sleeps instead of stealing issue slots from
// the walkers still running on its SM).
__device__ int64_t lookback(const Work &W, uint64_t g, uint32_t &sb_prev) {
    const int lane = lane_id();
    const uint64_t grp = g / LB_GROUP;
    const uint64_t g0 = grp * LB_GROUP;
    uint64_t k0 = 0;      // groups [0, k0) are summed into `done`
    int64_t done = 0;     // per-lane partial sum of confirmed groups
    bool own_ok = false;
    int64_t own = 0;
    uint32_t sbp = 0;
    uint32_t sleep_ns = SLEEP0;
    for (;;) {
        // groups [k0, grp), 32 per step, lane-parallel
        while (k0 < grp) {
            const uint64_t k = k0 + lane;
            unsigned long long wd = 0;
            bool ok = true;
            if (k < grp) {
                wd = ld_relaxed_u64(W.grp + k) + 1ull;  // groups before g's are full (LB_GROUP members)
                ok = (wd >> 48) == (unsigned long long)LB_GROUP;
            }
            const uint32_t bad = __ballot_sync(0xFFFFFFFFu, !ok);
            const uint32_t nvalid = (uint32_t)(grp - k0 < 32 ? grp - k0 : 32);
            const uint32_t ready = bad ? (uint32_t)(__ffs(bad) - 1) : nvalid;  // leading ready groups
            if ((uint32_t)lane < ready) done += (int64_t)(wd & LB_LOW48) - (int64_t)(LB_GROUP * LB_BIAS);
            k0 += ready;
            if (ready < nvalid) break;
        }
        if (!own_ok) {
            bool ok = true;
            own = 0;
            if (g0 + lane < g) {
                const unsigned long long wd = ld_relaxed_u64(W.status + g0 + lane);
                ok = (wd & ST_MASK) == ST_AGG;
                own = seg_a(wd);
                if (g0 + lane == g - 1) sbp = seg_sb(wd);
            } else if (lane == 31 && g0 == g) {  // g-1 ends the previous group
                const unsigned long long wd = ld_relaxed_u64(W.status + g - 1);
                ok = (wd & ST_MASK) == ST_AGG;
                sbp = seg_sb(wd);
            }
            own_ok = __all_sync(0xFFFFFFFFu, ok);
        }
        if (k0 == grp && own_ok) {
            int64_t sum = done + own;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
            sb_prev = __reduce_or_sync(0xFFFFFFFFu, sbp);  // only one lane holds it
            return sum;
        }
        __nanosleep(sleep_ns);
        if (sleep_ns < SLEEPMAX) sleep_ns <<= 1;
    }
}

template <int ALGO>
__global__ void __launch_bounds__(1024) k_fixup(Geometry G, Work W, uint64_t *d_count, uint64_t *file_out,
                                                uint64_t *bounds, uint64_t cap);

template <int ALGO, bool TM, int STG, bool FUSE, int SPM>
__device__ __forceinline__ void speculate_segment(const Geometry &G, Work &W, uint64_t g, uint64_t nsegs, uint8_t *wbase,
                                  uint64_t *bounds, uint64_t cap, uint64_t *d_count, int fused,
                                  int64_t pre_n = -1);

template <int ALGO>
__device__ int64_t t_coop_index(const Geometry &G, Work &W, uint64_t g, uint8_t *rings);

// K1.  One warp per segment (CTAs take segment groups in ticket order).  In
// the common case the fused look-back writes the output and k_fixup (launched
// behind it with PDL) only checks that it did.
// TM: the variant that tries the transfer tables (saturated streams); the
// other one carries none of their code, so the common path keeps its registers.
// NW warps per CTA with rings of 2 x STG bytes; FUSE: carries the fused
// look-back and write (the batch instance: BATCH_WARPS, BATCH_STAGE, no fused write).
template <int ALGO, bool TM, int NW = SPEC_WARPS, int STG = STAGE, bool FUSE = true, int SPM = 2>
__global__ void __launch_bounds__(NW * 32, SPEC_CTAS_PER_SM) k_speculate(Geometry G, Work W, uint64_t *bounds,
                                                                  uint64_t cap, uint64_t *d_count, int fused,
                                                                  int spw) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t s_ticket;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) stamp(TM_SPEC_BEGIN);
    if (gate0_shut(G.gate0)) return;
    pdl_wait();  // the reset of the published lists has completed
    if (G.gate && *G.gate == 0) return;  // the K-phase pipeline produced the output
    if (threadIdx.x == 0) {
        stamp(TM_SPEC_WAITED);
        s_ticket = atomicAdd(W.ctrl, 1u) + 1u;  // counter starts at ~0
    }
    __syncthreads();
    const uint64_t nsegs = total_segs(G, W);
    // spw segments per CTA (contiguous, so every predecessor is in this or an
    // earlier ticket); fewer than SPEC_WARPS spread a small input over the SMs.
    // spw = 0 (a batch): every warp takes segments one at a time from a global
    // ticket (segments of very different sizes; earlier segments are always
    // taken first, and without the fused write no warp waits on another).
    auto ticket = [&]() -> uint64_t {
        uint32_t t = 0;
        if (lane_id() == 0) t = atomicAdd(W.ctrl + DYN_TICKET, 1u) + 1u;  // counter starts at ~0
        return __shfl_sync(0xFFFFFFFFu, t, 0);
    };
    // a batch: tickets take the listed long segments, largest class first, then
    // every other segment in order (a listed one met there is skipped)
    auto next_seg = [&]() -> uint64_t {
        for (;;) {
            uint64_t t = ticket();
            const uint64_t total = G.total;
            for (int b = LPT_CLASSES - 1; b >= 0; --b) {
                const uint64_t c = (uint64_t)(W.tnx[b] + 1u);
                if (t < c) return W.lpt[lpt_base(total, b) + t];
                t -= c;
            }
            if (t >= nsegs || ((W.tblk[t >> 5] >> (t & 31)) & 1u)) return t;
        }
    };
    uint64_t g = spw == 0 ? next_seg() : (uint64_t)s_ticket * spw + warp;
    int64_t pre_n = -1;
    if constexpr (TM) {
        if (spw == 1) {  // one segment per CTA: its 16 warps build the index together
            if ((uint64_t)s_ticket >= nsegs) return;  // uniform across the CTA
            pre_n = t_coop_index<ALGO>(G, W, (uint64_t)s_ticket, align_smem(smem));
        }
    }
    if (spw != 0 && warp >= spw) return;
    constexpr int RS = Ring<STG>::SMEM;
    // the warp's ring: kept in a register (opaque to the compiler), so that the
    // walk does not rebuild it (thread index, alignment, multiply) at every use
    uint8_t *ring = align_smem(smem) + warp * RS;
    if (CDC_RING_OPAQUE) asm volatile("" : "+l"(ring));
    uint64_t *fetch = reinterpret_cast<uint64_t *>(ring + Ring<STG>::BYTES) + FETCH_SLOT;
    if (lane_id() == 0) *fetch = 0;
    while (g < nsegs) {  // one call site, so the walker is inlined once
        speculate_segment<ALGO, TM, STG, FUSE, SPM>(G, W, g, nsegs, ring, bounds, cap, d_count,
                                               FUSE ? fused : 0, pre_n);
        if (spw != 0) break;
        g = next_seg();
    }
    if (lane_id() == 0 && *fetch) atomicAdd(W.fetched, (unsigned long long)*fetch);
    if (lane_id() == 0) stamp(TM_SPEC_END);
}

#include "cdc_tables.cuh"  // T-mode: transfer tables for saturated streams

template <int ALGO, bool TM, int STG, bool FUSE, int SPM>
__device__ __forceinline__ void speculate_segment(const Geometry &G, Work &W, uint64_t g, uint64_t nsegs, uint8_t *wbase,
                                  uint64_t *bounds, uint64_t cap, uint64_t *d_count, int fused,
                                  int64_t pre_n) {
    if constexpr (!FUSE) fused = 0;
    const int lane = lane_id();
    static_assert(!TM || STG == STAGE, "the transfer tables use the default ring");
    WarpRing R{wbase, reinterpret_cast<uint64_t *>(wbase + Ring<STG>::BYTES)};

    SpecEmit em;
    em.G = &G;
    em.W = &W;
    em.I = seg_info(G, W, g);
    em.list = W.list + list_off(W, g);
    em.halo = W.halo + g * W.cap_halo;
    em.pub = W.pub + g;
    em.cnt = 1;
    em.hcnt = 0;
    em.sj = SJ_UNSYNCED;
    em.sa = em.sb = 0;
    em.lp.reset();
    em.published = false;
    if (lane == 0) st_relaxed_u32(em.list, 0u);  // the speculative chain starts at the segment's first byte
    unsigned long long *tm = g_timing ? g_timing + TM_STAMPS : nullptr;
    em.tbody = tm ? tm + TM_PER_SEG * g + 1 : nullptr;
    if (tm && lane == 0) tm[TM_PER_SEG * g] = globaltimer();
    const uint8_t *fbase = G.data + em.I.foff;
    if constexpr (TM) {  // transfer tables first: on a saturated stream no byte walk is needed
        if (t_attempt<ALGO>(G, W, g, nsegs, em.I, R.buf, fbase, bounds, cap, d_count, pre_n)) {
            if (lane == 0) {  // for cdc_stats: a table segment has no halo
                W.cnt[g] = 0;
                W.hcnt[g] = 0;
                W.sj[g] = SJ_TABLE;
                if (tm) tm[TM_PER_SEG * g + 3] = globaltimer();
            }
            return;
        }
    }
    int64_t read_end = (g == em.I.last) ? (int64_t)em.I.Lf
                                        : em.I.seg_end + (int64_t)G.Hmax + (int64_t)G.max_size;
    // the segment's head is read again by the previous segment's halo walk: keep it in L2
    const L2Pol pol{l2_evict_first_policy(), l2_evict_last_policy(), em.I.p + (int64_t)HEAD_KEEP};
    walk_chain<ALGO, STG, SPM>(G.sparse != 0, R, fbase, (int64_t)em.I.Lf, em.I.p, read_end, G.w, G.max_size, pol, em);
    em.publish();
    if (tm && lane == 0) {
        tm[TM_PER_SEG * g + 2] = globaltimer();
        tm[TM_PER_SEG * g + 4] = smid() | ((unsigned long long)em.hcnt << 32);
    }

    // ---- common case, fused resolve + write: the chain met the next segment's
    //      chain (or ended the file); anything else defers to k_fixup
    fused = fused && nsegs <= LB_MAX_SEGS;
    const bool normal = fused && (em.sj == SJ_LAST || em.sj == (int32_t)(g + 1));
    const uint32_t tail = em.sj == SJ_LAST ? 0u : em.sa;
    const uint32_t sb = normal && em.sj != SJ_LAST ? em.sb : 0u;
    const int64_t a = (int64_t)em.cnt + tail - sb;
    if (lane == 0) {
        W.cnt[g] = em.cnt;
        W.hcnt[g] = em.hcnt;
        W.sj[g] = em.sj;
        W.sa[g] = em.sa;
        W.sb[g] = em.sb;
        if (!normal) atomicAnd(W.ctrl + 1, 0u);  // the fast path's output is void
        if (em.sj == SJ_UNSYNCED) atomicAnd(W.ctrl + 2, 0u);  // (batch_resolve needs every halo decided)
    }
    // stage this segment's chain starts (list, then the halo tail) in the ring's
    // shared memory as offsets from p, so the write after the look-back needs no
    // global round trip (falls back to the global lists when they do not fit)
    uint32_t *stg = reinterpret_cast<uint32_t *>(wbase);
    const uint32_t nst = em.cnt + tail;
    const bool staged = nst <= (uint32_t)(Ring<STG>::BYTES / 4);
    if (fused && normal && staged) {
        const uint32_t hoff = (uint32_t)(em.I.seg_end - em.I.p);
        for (uint32_t i = lane; i < nst; i += 32)
            stg[i] = i < em.cnt ? ld_relaxed_u32(em.list + i) : hoff + em.halo[i - em.cnt];
    }
    if (fused) publish_agg(W, g, nsegs, a, sb);
    pdl_trigger();  // k_fixup may launch; it waits for this grid's completion
    if (!fused) return;
    uint32_t entry = 0;
    const int64_t excl = g == 0 ? 0 : lookback(W, g, entry);
    if (!normal) return;
    // entry(g) = sb(g-1), carried in segment g-1's status word
    if (g == em.I.first) entry = 0;
    const int64_t off = excl + entry;                     // output index of list[entry]
    const int64_t A = (int64_t)em.cnt - entry;            // true starts from this segment's list
    const int64_t n = A + tail;
    if (A < 0 || off < 0) {  // inconsistent (cannot happen when every segment is normal)
        if (lane == 0) atomicAnd(W.ctrl + 1, 0u);
        return;
    }
    __syncwarp();
    if (lane == 0) W.seg_out[g] = (uint64_t)off;
    for (int64_t i = lane; i < n; i += 32) {
        uint64_t v;
        if (staged) v = (uint64_t)em.I.p + stg[entry + i];
        else v = i < A ? (uint64_t)em.I.p + em.list[entry + i] : (uint64_t)em.I.seg_end + em.halo[i - A];
        const uint64_t q = (uint64_t)off + i;
        if (g == em.I.first && i == 0) continue;  // the file's first start (0) is not a boundary
        if (q - 1 < cap) bounds[q - 1] = v;
    }
    if (tm && lane == 0) tm[TM_PER_SEG * g + 3] = globaltimer();
    if (em.sj == SJ_LAST && lane == 0) {
        const uint64_t q = (uint64_t)(off + n) - 1;  // a file's last boundary is its length
        if (q < cap) bounds[q] = em.I.Lf;
        if (g == nsegs - 1) {
            *d_count = (uint64_t)(off + n);
            W.seg_out[nsegs] = (uint64_t)(off + n);
        }
    }
}

// ------------------------------------------------------------------ K2 walker emit
struct WalkEmit {
    const Geometry *G;
    const Work *W;
    SegInfo I;        // segment whose chain is being continued
    uint32_t *p32;    // slice of pool (entries relative to seg_end) ...
    uint64_t *p64;    // ... or pool B (file-relative entries)
    uint64_t base;    // first slot of this walker
    uint64_t lim;     // end of its slots
    uint64_t n;       // entries written
    int32_t sj;
    uint32_t sb;
    ListProbe lp;
    bool overflow;

    __device__ bool boundary(int64_t e) {
        int64_t j;
        uint32_t idx = 0;
        const int r = lp.probe(*W, I, e, j, idx);
        if (r == 1) {
            sj = (int32_t)j;
            sb = idx;
            return true;
        }
        if (base + n >= lim) {
            overflow = true;
            return true;
        }
        if (lane_id() == 0) {
            if (p32) p32[base + n] = (uint32_t)(e - I.seg_end);
            else p64[base + n] = (uint64_t)e;
        }
        ++n;
        return false;
    }
    __device__ bool in_halo() const { return false; }
    __device__ void end() { sj = SJ_STREAM_END; }
    __device__ void exhausted(int64_t) { sj = SJ_STREAM_END; }
};

// block-wide exclusive scan helper (1024 threads)
__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t &total, uint64_t *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t s = lane < nw ? scratch[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= o) s += y;
        }
        scratch[32 + lane] = s;
    }
    __syncthreads();
    uint64_t warp_prefix = warp ? scratch[32 + warp - 1] : 0;
    total = scratch[32 + nw - 1];
    __syncthreads();
    return warp_prefix + x - v;
}

// Decoupled look-back over tiles (k_seg_prefix, the batch resolve): a word is
// a flag (top two bits) and a non-negative 62-bit value; k_reset leaves ~0 =
// not ready.  Every word is self-contained, so relaxed accesses suffice.
constexpr unsigned long long TL_AGG = 1ull << 62;  // the tile's own total
constexpr unsigned long long TL_INC = 2ull << 62;  // the inclusive prefix through the tile
constexpr unsigned long long TL_VAL = (1ull << 62) - 1;
__device__ __forceinline__ void tile_publish(unsigned long long *w, unsigned long long flag, uint64_t v) {
    asm volatile("st.relaxed.gpu.u64 [%0], %1;" ::"l"(w), "l"(flag | (v & TL_VAL)) : "memory");
}
// All 32 lanes: the exclusive prefix of tile t from the words st[k * stride],
// k < t, read 32 at a time from t-1 downwards until an inclusive one.
__device__ uint64_t tile_lookback(const unsigned long long *st, uint64_t stride, uint64_t t) {
    const int lane = lane_id();
    uint64_t excl = 0;
    int64_t k = (int64_t)t - 1;
    while (k >= 0) {
        const int64_t i = k - lane;
        const unsigned long long wd = i >= 0 ? ld_relaxed_u64(st + (uint64_t)i * stride) : TL_INC;
        const unsigned long long fl = wd & ~TL_VAL;
        const uint32_t inc = __ballot_sync(0xFFFFFFFFu, fl == TL_INC);
        const uint32_t bad = __ballot_sync(0xFFFFFFFFu, fl != TL_INC && fl != TL_AGG);
        const int fi = inc ? __ffs(inc) - 1 : 31;  // lanes 0..fi are needed
        const uint32_t need = fi == 31 ? 0xFFFFFFFFu : ((2u << fi) - 1u);
        if (bad & need) {
            __nanosleep(100);
            continue;
        }
        uint64_t v = (lane <= fi && i >= 0) ? (uint64_t)(wd & TL_VAL) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        excl += v;
        if (inc) break;
        k -= 32;
    }
    return excl;
}

constexpr int RPT = 8;           // resolve_block: consecutive segments per thread in the count scan
constexpr int FIX_WALKERS = 8;   // resolve_block: parallel fix-up walkers (one smem ring each)
constexpr int FIX_STAGE = (FIX_WALKERS - 2) * RING_SMEM / 12;  // exceptional segments staged per round (+ one ring)
constexpr int FIX_SMEM = FIX_WALKERS * RING_SMEM + 128;  // k_fixup dynamic shared memory

// Where the true chain goes after exceptional segment g (when g is on it):
// 0 = into the next segment (no jump), TGT_WALK = not known yet (a fix-up walk
// must continue the chain), else the first segment after the jump.
constexpr uint32_t TGT_WALK = 0xFFFFFFFFu;
__device__ __forceinline__ uint32_t exc_target(const Geometry &G, const Work &W, uint64_t g) {
    const int32_t sj = W.sj[g];
    if (sj == SJ_UNSYNCED) return TGT_WALK;
    if (sj == SJ_STREAM_END) {
        uint64_t fa, fb;
        seg_first_of(G, W, file_of_seg(G, W, g), fa, fb);
        return (uint32_t)fb;  // past the file's last segment
    }
    if (sj == SJ_LAST || sj == (int32_t)(g + 1)) return 0;
    return (uint32_t)sj;
}

// Re-check the halo of segment g (left undecided by K1) against the complete
// lists: 32 halo entries at a time, each lane binary-searching the list of the
// segment its entry lies in; the first entry found is the sync point.
__device__ void recheck_halo(const Geometry &G, Work &W, uint64_t g) {
    const int lane = lane_id();
    SegInfo I = seg_info(G, W, g);
    const uint32_t hc = W.hcnt[g];
    for (uint32_t i0 = 0; i0 < hc; i0 += 32) {
        const uint32_t i = i0 + lane;
        bool found = false;
        int64_t j = 0;
        uint32_t idx = 0;
        if (i < hc) {
            const int64_t e = I.seg_end + (int64_t)W.halo[g * W.cap_halo + i];
            int64_t pj;
            j = seg_of_pos(I, e, G.S, pj);
            const uint32_t r = (uint32_t)(e - pj);
            const uint32_t *lst = W.list + list_off(W, (uint64_t)j);
            uint32_t lo = 0, hi = W.cnt[j];
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (lst[mid] < r) lo = mid + 1;
                else hi = mid;
            }
            found = lo < W.cnt[j] && lst[lo] == r;
            idx = lo;
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, found);
        if (bal) {
            const int L = __ffs(bal) - 1;
            if (lane == L) {
                W.sj[g] = (int32_t)j;
                W.sa[g] = i;
                W.sb[g] = idx;
            }
            return;
        }
    }
}

// K2: one CTA.  Common case (every segment's chain re-synchronised with the
// next segment's): two coalesced passes -- classify, then per-segment output
// counts and their exclusive scan.  Exceptional segments (a sync target other
// than the next segment, or an undecided halo) take the serial path.
template <int ALGO>
__device__ void resolve_block(const Geometry &G, Work &W, uint64_t *d_count, uint64_t *file_out) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t scratch[64];
    __shared__ uint64_t s_carry;
    __shared__ int s_flags;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const uint64_t nsegs = total_segs(G, W);
    if (nsegs > 0 && W.ctrl[1] != 0u) {
        // k_speculate's fused look-back produced the output: only the per-file offsets remain
        const uint64_t nf = G.file_off == nullptr ? 0 : G.nfiles;
        for (uint64_t f = tid; f <= nf && G.file_off != nullptr; f += blockDim.x) {
            const uint64_t sf = W.seg_first[f];
            file_out[f] = (sf >= nsegs) ? W.seg_out[nsegs] : W.seg_out[sf];
        }
        return;
    }

    // 1. classify (32 consecutive segments per warp step, coalesced); re-check
    //    undecided halos now that every list is complete
    if (tid == 0) s_flags = 0;
    __syncthreads();
    int fl = 0;
    for (uint64_t g0 = (uint64_t)warp * 32; g0 < nsegs; g0 += (uint64_t)nwarps * 32) {
        const uint64_t g = g0 + lane;
        const int32_t sj0 = g < nsegs ? W.sj[g] : SJ_LAST;
        uint32_t un = __ballot_sync(0xFFFFFFFFu, sj0 == SJ_UNSYNCED);
        while (un) {
            const int L = __ffs(un) - 1;
            un &= un - 1;
            recheck_halo(G, W, g0 + L);
        }
        __syncwarp();
        const int32_t sj = g < nsegs ? W.sj[g] : SJ_LAST;
        if (sj != SJ_LAST && sj != (int32_t)(g + 1)) fl = 1;
    }
    if (fl) atomicOr(&s_flags, 1);
    __syncthreads();
    const bool exc = s_flags != 0;

    if (exc) {
        for (uint64_t g = tid; g < nsegs; g += blockDim.x) {
            W.skipped[g] = 0;
            W.wcnt[g] = 0;
            W.ocnt[g] = 0;
            W.jump_entry[g] = 0;
        }
        if (tid == 0) {
            W.misc[2] = 0;  // ranges
            W.misc[3] = 0;  // overflow
            W.misc[5] = 0;  // reach
        }
        __syncthreads();
        // 2. compact the exceptional segments in order
        if (tid == 0) s_carry = 0;
        __syncthreads();
        for (uint64_t base = 0; base < nsegs; base += blockDim.x) {
            uint64_t g = base + tid;
            uint64_t flag = 0;
            if (g < nsegs) {
                int32_t sj = W.sj[g];
                flag = (sj != SJ_LAST && sj != (int32_t)(g + 1)) ? 1 : 0;
            }
            uint64_t tot;
            uint64_t pos = block_exclusive_scan(flag, tot, scratch) + s_carry;
            if (flag && pos < W.exc_cap) W.exc[pos] = (uint32_t)g;
            __syncthreads();
            if (tid == 0) s_carry += tot;
            __syncthreads();
        }
        const uint64_t n_exc = s_carry;

        // 3a. unsynced halos, continued in parallel (FIX_WALKERS warps, one ring each)
        //     from their last recorded start until they meet a later segment's chain;
        //     walker g writes into its own pool slice and, should the slice fill up,
        //     leaves the segment unsynced for the serial pass (3b)
        if (warp < FIX_WALKERS) {
            uint8_t *rb = align_smem(smem) + warp * RING_SMEM;
            WarpRing R{rb, reinterpret_cast<uint64_t *>(rb + RING_BYTES)};
            for (uint64_t x = warp; x < n_exc && x < W.exc_cap; x += FIX_WALKERS) {
                const uint64_t g = W.exc[x];
                if (W.sj[g] != SJ_UNSYNCED) continue;
                SegInfo I = seg_info(G, W, g);
                WalkEmit em;
                em.G = &G;
                em.W = &W;
                em.I = I;
                em.p32 = W.pool;
                em.p64 = nullptr;
                em.base = g * W.cap_halo;
                em.lim = em.base + W.cap_halo;
                em.n = 0;
                em.sj = SJ_STREAM_END;
                em.sb = 0;
                em.lp.reset();
                em.overflow = false;
                const uint32_t hc = W.hcnt[g];
                const int64_t last = hc ? I.seg_end + (int64_t)W.halo[g * W.cap_halo + hc - 1]
                                        : I.p + (int64_t)W.list[list_off(W, g) + W.cnt[g] - 1];
                walk_chain<ALGO>(G.sparse != 0, R, G.data + I.foff, (int64_t)I.Lf, last, (int64_t)I.Lf, G.w, G.max_size,
                                stream_policy(), em);
                if (lane == 0) {
                    W.sj[g] = em.overflow ? SJ_UNSYNCED : em.sj;
                    W.sa[g] = hc;
                    W.sb[g] = em.sb;
                    W.wcnt[g] = (uint32_t)em.n;
                    W.woff[g] = em.base;
                }
            }
        }
        __syncthreads();

        // 3b. the true chain through the exceptional segments, in order (warp 0), from
        //     jump targets staged in shared memory; a segment still unsynced (its
        //     slice filled up) is continued here, serially, into pool B
        uint32_t *s_exc = reinterpret_cast<uint32_t *>(align_smem(smem));
        uint32_t *s_tgt = s_exc + FIX_STAGE;
        uint32_t *s_sb = s_tgt + FIX_STAGE;  // sb of the segment, or ~0 when it has no sync target
        uint64_t reach = 0, nrng = 0, poolb_used = 0;
        bool overflow = false;
        for (uint64_t x0 = 0; x0 < n_exc && x0 < W.exc_cap; x0 += FIX_STAGE) {
            const uint64_t m = (n_exc - x0 < FIX_STAGE ? n_exc - x0 : FIX_STAGE);
            __syncthreads();
            for (uint64_t i = tid; i < m; i += blockDim.x) {
                const uint64_t g = W.exc[x0 + i];
                s_exc[i] = (uint32_t)g;
                s_tgt[i] = exc_target(G, W, g);
                s_sb[i] = W.sj[g] >= 0 ? W.sb[g] : 0xFFFFFFFFu;
            }
            __syncthreads();
            if (warp == 0) {
                for (uint64_t i = 0; i < m; ++i) {
                    const uint64_t g = s_exc[i];
                    if (g < reach) continue;  // skipped by an earlier jump: not on the true chain
                    uint32_t target = s_tgt[i];
                    if (target == TGT_WALK) {  // continue the chain from the end of its slice
                        SegInfo I = seg_info(G, W, g);
                        uint8_t *rb = align_smem(align_smem(smem) + 3 * FIX_STAGE * 4);  // after the staged arrays
                        WarpRing R{rb, reinterpret_cast<uint64_t *>(rb + RING_BYTES)};
                        WalkEmit em;
                        em.G = &G;
                        em.W = &W;
                        em.I = I;
                        em.p32 = nullptr;
                        em.p64 = W.poolb;
                        em.base = poolb_used;
                        em.lim = W.poolb_cap;
                        em.n = 0;
                        em.sj = SJ_STREAM_END;
                        em.sb = 0;
                        em.lp.reset();
                        em.overflow = false;
                        const uint32_t wc = W.wcnt[g];
                        const int64_t last = I.seg_end + (int64_t)W.pool[W.woff[g] + wc - 1];
                        walk_chain<ALGO>(G.sparse != 0, R, G.data + I.foff, (int64_t)I.Lf, last, (int64_t)I.Lf, G.w, G.max_size,
                                        stream_policy(), em);
                        overflow |= em.overflow;
                        if (lane == 0) {
                            W.sj[g] = em.sj;
                            W.sb[g] = em.sb;
                            W.ocnt[g] = (uint32_t)em.n;
                            W.ooff[g] = em.base;
                        }
                        poolb_used += em.n;
                        __syncwarp();
                        target = exc_target(G, W, g);
                        if (lane == 0) s_sb[i] = W.sj[g] >= 0 ? W.sb[g] : 0xFFFFFFFFu;
                        __syncwarp();
                    }
                    if (target == 0) continue;  // met the next segment's chain: no skip
                    if (lane == 0) {
                        W.ranges[2 * nrng] = (uint32_t)(g + 1);
                        W.ranges[2 * nrng + 1] = target;
                        if (s_sb[i] != 0xFFFFFFFFu) W.jump_entry[target] = s_sb[i];
                    }
                    ++nrng;
                    reach = target;
                }
            }
        }
        if (warp == 0 && lane == 0) {
            W.misc[2] = (uint32_t)nrng;
            W.misc[3] = (overflow || n_exc > W.exc_cap) ? 1u : 0u;
        }
        __syncthreads();

        // 4. mark segments the true chain jumps over
        const uint32_t nranges = W.misc[2];
        for (uint32_t r = warp; r < nranges; r += nwarps) {
            const uint32_t a = W.ranges[2 * r], b = W.ranges[2 * r + 1];
            for (uint32_t g = a + lane; g < b; g += 32) W.skipped[g] = 1;
        }
        __syncthreads();
    }
    if (tid == 0) W.misc[4] = exc ? 1u : 0u;  // the writers: skipped / wcnt are valid only if set

    // 5. per-segment output counts (RPT consecutive segments per thread) and their exclusive scan
    if (tid == 0) s_carry = 0;
    __syncthreads();
    const uint64_t TILE = (uint64_t)blockDim.x * RPT;
    for (uint64_t base = 0; base < nsegs; base += TILE) {
        uint32_t nloc[RPT];
        uint64_t tsum = 0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const uint64_t g = base + (uint64_t)tid * RPT + i;
            uint32_t n = 0;
            if (g < nsegs && !(exc && W.skipped[g])) {
                const bool first = G.file_off == nullptr ? g == 0 : W.seg_first[W.seg_file[g]] == g;
                uint32_t e = 0;
                if (!first) e = (exc && W.skipped[g - 1]) ? W.jump_entry[g] : W.sb[g - 1];
                const int32_t sj = W.sj[g];
                const uint32_t tail = sj == SJ_STREAM_END ? W.hcnt[g] : (sj >= 0 ? W.sa[g] : 0u);
                W.entry[g] = e;
                W.tail[g] = tail;
                n = (W.cnt[g] - e) + tail + (exc ? W.wcnt[g] + W.ocnt[g] : 0u);
            }
            nloc[i] = n;
            tsum += n;
        }
        uint64_t tot;
        uint64_t pos = block_exclusive_scan(tsum, tot, scratch) + s_carry;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const uint64_t g = base + (uint64_t)tid * RPT + i;
            if (g < nsegs) W.seg_out[g] = pos;
            pos += nloc[i];
        }
        __syncthreads();
        if (tid == 0) s_carry += tot;
        __syncthreads();
    }
    const uint64_t total = s_carry;
    if (tid == 0) {
        W.seg_out[nsegs] = total;
        *d_count = total;
    }
    // 6. per-file output offsets
    const uint64_t nf = G.file_off == nullptr ? 1 : G.nfiles;
    for (uint64_t f = tid; f <= nf; f += blockDim.x) {
        uint64_t sf = (G.file_off == nullptr) ? (f == 0 ? 0 : nsegs) : W.seg_first[f];
        file_out[f] = (sf >= nsegs) ? total : W.seg_out[sf];
    }
}

// ------------------------------------------------------------------ K3 write
__device__ void write_segment(const Geometry &G, const Work &W, const uint64_t *file_out, uint64_t *bounds,
                              uint64_t cap, uint64_t g) {
    const int lane = lane_id();
    SegInfo I = seg_info(G, W, g);
    const uint64_t fo = file_out[I.f];
    if (g == I.first && lane == 0 && I.Lf > 0) {
        const uint64_t q = file_out[I.f + 1] - 1;  // a stream's last boundary is its length
        if (q < cap) bounds[q] = I.Lf;
    }
    const bool exc = W.misc[4] != 0;
    if (exc && W.skipped[g]) return;
    const uint32_t e = W.entry[g], cnt = W.cnt[g], tail = W.tail[g], wc = exc ? W.wcnt[g] : 0u;
    const uint32_t oc = exc ? W.ocnt[g] : 0u;
    const uint64_t A = cnt - e, n = A + tail + wc + oc, base = W.seg_out[g];
    const uint32_t *lst = W.list + list_off(W, g);
    const uint32_t *hl = W.halo + g * W.cap_halo;
    for (uint64_t i = lane; i < n; i += 32) {
        uint64_t v;
        if (i < A) v = (uint64_t)I.p + lst[e + i];
        else if (i < A + tail) v = (uint64_t)I.seg_end + hl[i - A];
        else if (i < A + tail + wc) v = (uint64_t)I.seg_end + W.pool[W.woff[g] + (i - A - tail)];
        else v = W.poolb[W.ooff[g] + (i - A - tail - wc)];
        const uint64_t q = base + i;
        if (q == fo) continue;  // the stream's first start (0) is not a boundary
        if (q - 1 < cap) bounds[q - 1] = v;
    }
}

// A batch whose every halo was decided (it met a later segment's chain of its
// file, or reached the file's end; k_speculate clears ctrl[CT_BATCH_NORMAL]
// otherwise).  Phase 0: one thread per file follows the true chain through
// the file's segments (segment g's halo leads to its sync target sj(g) with
// entry sb(g); segments it jumps over, and every segment after a halo that
// reached the file's end, are skipped).  Phase 1: every CTA scans tiles of
// BR_RPT x 1024 segments' output counts, chained by a decoupled look-back.
// Phase 2: once every tile is done, every CTA writes its share of the
// segments' boundaries and the per-file offsets.  Work is taken from tickets
// by running CTAs, so the waits for a phase cannot block on a CTA that has
// not started.
constexpr int BR_RPT = 2;
constexpr int CT_BATCH_NORMAL = 2, CT_BR_TICKET = 7, CT_BR_DONE = 8, CT_SP_TICKET = 6;
constexpr int CT_BR0_TICKET = 10, CT_BR0_DONE = 11;  // (batch only: T-mode, which uses them, is single-stream)
__device__ void batch_resolve(const Geometry &G, Work &W, uint64_t nsegs, uint64_t *d_count, uint64_t *file_out,
                              uint64_t *bounds, uint64_t cap) {
    __shared__ uint64_t scratch[64];
    __shared__ uint64_t s_ex;
    __shared__ uint32_t s_t;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // phase 0: the true chain through each file's segments
    const uint64_t nblk0 = (G.nfiles + blockDim.x - 1) / blockDim.x;
    for (;;) {
        if (tid == 0) s_t = atomicAdd(W.ctrl + CT_BR0_TICKET, 1u) + 1u;  // the counter starts at ~0
        __syncthreads();
        const uint64_t t = s_t;
        __syncthreads();
        if (t >= nblk0) break;  // uniform across the CTA
        const uint64_t f = t * blockDim.x + tid;
        if (f < G.nfiles) {
            const uint64_t a = W.seg_first[f], b = W.seg_first[f + 1];
            uint32_t e = 0;
            uint64_t h = a;
            while (h < b) {
                W.entry[h] = e;
                W.skipped[h] = 0;
                const int32_t sj = W.sj[h];
                if (sj == SJ_LAST) {
                    W.tail[h] = 0;
                    break;
                }
                if (sj < 0) {  // SJ_STREAM_END: the halo carries the chain to the file's end
                    W.tail[h] = W.hcnt[h];
                    for (uint64_t k = h + 1; k < b; ++k) W.skipped[k] = 1;
                    break;
                }
                W.tail[h] = W.sa[h];
                for (uint64_t k = h + 1; k < (uint64_t)sj; ++k) W.skipped[k] = 1;
                e = W.sb[h];
                h = (uint64_t)sj;
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(W.ctrl + CT_BR0_DONE, 1u);
        }
    }
    if (tid == 0) {
        while (ld_acquire_u32(W.ctrl + CT_BR0_DONE) + 1u != (uint32_t)nblk0) __nanosleep(256);
    }
    __syncthreads();
    const uint64_t BT = (uint64_t)blockDim.x * BR_RPT;
    const uint64_t ntiles = (nsegs + BT - 1) / BT;
    for (;;) {
        if (tid == 0) s_t = atomicAdd(W.ctrl + CT_BR_TICKET, 1u) + 1u;  // the counter starts at ~0
        __syncthreads();
        const uint64_t t = s_t;
        if (t >= ntiles) break;  // uniform across the CTA
        uint32_t nloc[BR_RPT];
        uint64_t sum = 0;
#pragma unroll
        for (int i = 0; i < BR_RPT; ++i) {
            const uint64_t g = t * BT + (uint64_t)tid * BR_RPT + i;
            uint32_t n = 0;
            if (g < nsegs && !W.skipped[g]) n = W.cnt[g] - W.entry[g] + W.tail[g];
            nloc[i] = n;
            sum += n;
        }
        uint64_t tot;
        uint64_t pos = block_exclusive_scan(sum, tot, scratch);  // (its barriers also order the read of s_t)
        if (warp == 0) {
            uint64_t ex = 0;
            if (t == 0) {
                if (lane == 0) tile_publish(W.grp, TL_INC, tot);
            } else {
                if (lane == 0) tile_publish(W.grp + t, TL_AGG, tot);
                ex = tile_lookback(W.grp, 1, t);
                if (lane == 0) tile_publish(W.grp + t, TL_INC, ex + tot);
            }
            if (lane == 0) s_ex = ex;
        }
        __syncthreads();
        pos += s_ex;
#pragma unroll
        for (int i = 0; i < BR_RPT; ++i) {
            const uint64_t g = t * BT + (uint64_t)tid * BR_RPT + i;
            if (g < nsegs) W.seg_out[g] = pos;
            pos += nloc[i];
        }
        if (t == ntiles - 1 && tid == 0) {
            W.seg_out[nsegs] = s_ex + tot;
            *d_count = s_ex + tot;
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(W.ctrl + CT_BR_DONE, 1u);
        }
    }
    if (tid == 0) {
        while (ld_acquire_u32(W.ctrl + CT_BR_DONE) + 1u != (uint32_t)ntiles) __nanosleep(256);
    }
    __syncthreads();
    // boundaries: each warp takes 32 consecutive segments; lane k loads segment
    // g0+k's record (32 records' dependent loads in flight together), then the
    // warp writes the 32 segments' boundaries one after another with all lanes
    const uint64_t nwg = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t g0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32; g0 < nsegs; g0 += nwg * 32) {
        const uint64_t g = g0 + lane;
        uint32_t n = 0, A = 0;
        uint64_t base = 0, fo = 0, p = 0, se = 0, lp = 0;
        if (g < nsegs && !W.skipped[g]) {  // (a skipped segment is never a file's first)
            const SegInfo I = seg_info(G, W, g);
            fo = W.seg_out[I.first];
            if (g == I.first && I.Lf > 0) {
                const uint64_t q = W.seg_out[I.last + 1] - 1;  // a file's last boundary is its length
                if (q < cap) bounds[q] = I.Lf;
            }
            const uint32_t e = W.entry[g];
            A = W.cnt[g] - e;
            n = A + W.tail[g];
            base = W.seg_out[g];
            p = (uint64_t)I.p;
            se = (uint64_t)I.seg_end;
            lp = list_off(W, g) + e;
        }
        for (int r = 0; r < 32; ++r) {
            const uint32_t rn = __shfl_sync(0xFFFFFFFFu, n, r);
            if (rn == 0) continue;
            const uint32_t rA = __shfl_sync(0xFFFFFFFFu, A, r);
            const uint64_t rb = __shfl_sync(0xFFFFFFFFu, base, r), rfo = __shfl_sync(0xFFFFFFFFu, fo, r);
            const uint64_t rp = __shfl_sync(0xFFFFFFFFu, p, r), rse = __shfl_sync(0xFFFFFFFFu, se, r);
            const uint64_t rlp = __shfl_sync(0xFFFFFFFFu, lp, r);
            const uint32_t *hl = W.halo + (g0 + r) * W.cap_halo;
            for (uint32_t i = lane; i < rn; i += 32) {
                const uint64_t v = i < rA ? rp + W.list[rlp + i] : rse + hl[i - rA];
                const uint64_t q = rb + i;
                if (q == rfo) continue;  // the file's first start (0) is not a boundary
                if (q - 1 < cap) bounds[q - 1] = v;
            }
        }
    }
    // per-file output offsets
    const uint64_t total = W.seg_out[nsegs];
    for (uint64_t f = (uint64_t)blockIdx.x * blockDim.x + tid; f <= G.nfiles; f += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t sf = W.seg_first[f];
        file_out[f] = sf >= nsegs ? total : W.seg_out[sf];
    }
}

// K2 (fix-up, one launch): when k_speculate's fused fast path succeeded this
// exits at once (a batch still needs its per-file offsets, computed by the
// first CTA).  Otherwise the CTA that draws ticket 0 resolves the true chain
// (resolve_block: one CTA of 1024 threads) and releases a flag; every CTA then
// writes the boundaries of its 32 segments (one warp each).  Tickets make the
// waiting safe: the resolver is the first CTA to run.
template <int ALGO>
__global__ void __launch_bounds__(1024) k_fixup(Geometry G, Work W, uint64_t *d_count, uint64_t *file_out,
                                                uint64_t *bounds, uint64_t cap) {
    __shared__ uint32_t s_role;
    if (threadIdx.x == 0) stamp(TM_FIX_BEGIN);
    if (gate0_shut(G.gate0)) return;
    pdl_wait();  // k_speculate has completed and its writes are visible
    if (G.gate && *G.gate == 0) return;  // the K-phase pipeline produced the output
    if (threadIdx.x == 0) stamp(TM_FIX_WAITED);
    const uint64_t nsegs = total_segs(G, W);
    if (G.file_off != nullptr && nsegs > 0 && W.ctrl[CT_BATCH_NORMAL] != 0u) {
        batch_resolve(G, W, nsegs, d_count, file_out, bounds, cap);
        if (threadIdx.x == 0) stamp(TM_FIX_END);
        return;
    }
    const bool fast = nsegs > 0 && W.ctrl[1] != 0u;
    if (fast && G.file_off == nullptr) {
        if (threadIdx.x == 0) stamp(TM_FIX_END);
        return;
    }
    if (threadIdx.x == 0) s_role = atomicAdd(W.ctrl + 3, 1u) + 1u;  // counter starts at ~0
    __syncthreads();
    const uint32_t role = s_role;
    if (role == 0) {
        resolve_block<ALGO>(G, W, d_count, file_out);
        __syncthreads();
        if (threadIdx.x == 0) st_release_u64(reinterpret_cast<unsigned long long *>(W.ctrl + 4), 1ull);
    }
    if (fast) return;
    if (threadIdx.x == 0) {
        while (ld_acquire_u64(reinterpret_cast<const unsigned long long *>(W.ctrl + 4)) != 1ull) __nanosleep(256);
    }
    __syncthreads();
    for (uint64_t g = (uint64_t)role * 32 + (threadIdx.x >> 5); g < nsegs; g += (uint64_t)gridDim.x * 32)
        write_segment(G, W, file_out, bounds, cap, g);
}

#include "cdc_kphase.cuh"  // K-phase speculation: single streams with long windows
#include "cdc_dense.cuh"   // dense-index mode: small single streams saturated everywhere
#include "cdc_maxp.cuh"    // MAXP: local maxima in one pass, then the chain over them

// ------------------------------------------------------------------ K0 batch segment table
// Tiles of SP_THREADS x SP_RPT consecutive files, taken from a ticket by a
// small grid, chained by a decoupled look-back (tile_lookback).  Writes
// seg_first (first segment of each file), seg_file (segment -> file) and lofs
// (first list entry of each segment: a segment of len bytes gets
// len / (w+1) + 2 entries -- every chunk but a file's last is longer than w).
constexpr int SP_THREADS = 256, SP_RPT = 4;
__device__ __forceinline__ void block_exclusive_scan2(uint64_t &a, uint64_t &b, uint64_t &ta, uint64_t &tb,
                                                      uint64_t *scratch) {
    // scratch: 4 x 32 words
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t x = a, y = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, x, o), v = __shfl_up_sync(0xFFFFFFFFu, y, o);
        if (lane >= o) {
            x += u;
            y += v;
        }
    }
    if (lane == 31) {
        scratch[warp] = x;
        scratch[32 + warp] = y;
    }
    __syncthreads();
    if (warp == 0) {
        uint64_t sx = lane < nw ? scratch[lane] : 0, sy = lane < nw ? scratch[32 + lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, sx, o), v = __shfl_up_sync(0xFFFFFFFFu, sy, o);
            if (lane >= o) {
                sx += u;
                sy += v;
            }
        }
        scratch[64 + lane] = sx;
        scratch[96 + lane] = sy;
    }
    __syncthreads();
    const uint64_t px = warp ? scratch[64 + warp - 1] : 0, py = warp ? scratch[96 + warp - 1] : 0;
    ta = scratch[64 + nw - 1];
    tb = scratch[96 + nw - 1];
    __syncthreads();
    a = px + x - a;
    b = py + y - b;
}

// st: two look-back words per tile (segments, list entries), reset to ~0 by k_reset;
// ticket: ctrl[SP_TICKET] (reset to ~0)
__global__ void __launch_bounds__(SP_THREADS) k_seg_prefix(const uint64_t *file_off, uint64_t nfiles, uint64_t S,
                                                           uint64_t w1, uint64_t *seg_first, uint32_t *seg_file,
                                                           uint64_t *lofs, unsigned long long *st,
                                                           uint32_t *ticket, LptLists lpt) {
    __shared__ uint64_t scratch[128];
    __shared__ uint64_t s_ex[2];
    __shared__ uint32_t s_t;
    pdl_trigger();  // k_speculate may launch now; it waits for this grid's completion
    pdl_wait();     // k_reset has completed (look-back words and ticket)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t TILE = (uint64_t)SP_THREADS * SP_RPT;
    const uint64_t ntiles = (nfiles + TILE - 1) / TILE;
    if (nfiles == 0 && blockIdx.x == 0 && tid == 0) {
        seg_first[0] = 0;
        lofs[0] = 0;
    }
    for (;;) {
        if (tid == 0) s_t = atomicAdd(ticket, 1u) + 1u;  // the counter starts at ~0
        __syncthreads();
        const uint64_t t = s_t;
        if (t >= ntiles) break;  // uniform across the CTA
        const uint64_t f0 = t * TILE + (uint64_t)tid * SP_RPT;
        uint64_t ns = 0, nl = 0;
        for (int i = 0; i < SP_RPT; ++i) {
            const uint64_t f = f0 + i;
            if (f >= nfiles) break;
            const uint64_t len = file_off[f + 1] - file_off[f];
            const uint64_t n = nseg_of(len, S);
            ns += n;
            nl += len / w1 + 2 * n;  // sum over the file's segments of seg_len / w1 + 2 (floor of a sum >= sum of floors)
        }
        uint64_t ts, tl;
        block_exclusive_scan2(ns, nl, ts, tl, scratch);  // (its barriers also order the read of s_t)
        if (warp == 0) {
            uint64_t es = 0, el = 0;
            if (t == 0) {
                if (lane == 0) {
                    tile_publish(st, TL_INC, ts);
                    tile_publish(st + 1, TL_INC, tl);
                }
            } else {
                if (lane == 0) {
                    tile_publish(st + 2 * t, TL_AGG, ts);
                    tile_publish(st + 2 * t + 1, TL_AGG, tl);
                }
                es = tile_lookback(st, 2, t);
                el = tile_lookback(st + 1, 2, t);
                if (lane == 0) {
                    tile_publish(st + 2 * t, TL_INC, es + ts);
                    tile_publish(st + 2 * t + 1, TL_INC, el + tl);
                }
            }
            if (lane == 0) {
                s_ex[0] = es;
                s_ex[1] = el;
            }
        }
        __syncthreads();
        uint64_t ps = s_ex[0] + ns, pl = s_ex[1] + nl;
        for (int i = 0; i < SP_RPT; ++i) {
            const uint64_t f = f0 + i;
            if (f >= nfiles) break;
            const uint64_t len = file_off[f + 1] - file_off[f];
            const uint64_t n = nseg_of(len, S);
            seg_first[f] = ps;
            uint64_t used = 0;
            for (uint64_t k = 0; k < n; ++k) {  // segment -> file map and list offsets
                const uint64_t sl = (uint64_t)(seg_start(k + 1, n, len) - seg_start(k, n, len));
                seg_file[ps + k] = (uint32_t)f;
                lofs[ps + k] = pl + used;
                used += sl / w1 + 2;
                if (sl >> LPT_MIN_LOG2) {
                    const uint64_t g = ps + k;
                    int b = 63 - __clzll((long long)(sl >> LPT_MIN_LOG2));
                    b = b < LPT_CLASSES - 1 ? b : LPT_CLASSES - 1;
                    const uint32_t i = atomicAdd(lpt.cnt + b, 1u) + 1u;  // the counter starts at ~0
                    lpt.list[lpt_base(lpt.total, b) + i] = (uint32_t)g;
                    atomicAnd(lpt.map + (g >> 5), ~(1u << (g & 31)));
                }
            }
            ps += n;
            pl += len / w1 + 2 * n;
        }
        if (t == ntiles - 1 && tid == 0) {
            seg_first[nfiles] = s_ex[0] + ts;
            lofs[s_ex[0] + ts] = s_ex[1] + tl;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ chain API kernel
struct ChainEmit {
    uint64_t *out;
    uint64_t cap, n;
    int64_t stop, len;
    __device__ bool boundary(int64_t e) {
        if (lane_id() == 0 && n < cap) out[n] = (uint64_t)e;
        ++n;
        return e >= stop;
    }
    // the chain's last chunk ends at len: record len as its final position
    __device__ bool in_halo() const { return false; }
    __device__ void end() {
        if (lane_id() == 0 && n < cap) out[n] = (uint64_t)len;
        ++n;
    }
    __device__ void exhausted(int64_t) {}
};

template <int ALGO>
__global__ void __launch_bounds__(32) k_chain(const uint8_t *data, uint64_t len, uint64_t start, uint64_t stop,
                                              uint32_t w, uint64_t max_size, uint64_t *out, uint64_t cap,
                                              uint64_t *count, int sparse) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *rb = align_smem(smem);
    WarpRing R{rb, reinterpret_cast<uint64_t *>(rb + RING_BYTES)};
    ChainEmit em{out, cap, 0, (int64_t)stop, (int64_t)len};
    if (lane_id() == 0 && cap > 0) out[0] = start;
    em.n = 1;
    if (start < stop && start < len)
        walk_chain<ALGO>(sparse != 0, R, data, (int64_t)len, (int64_t)start, (int64_t)len, w, max_size, stream_policy(),
                         em);
    if (lane_id() == 0) *count = em.n;
}

// ------------------------------------------------------------------ cross-shard re-synchronisation
// First element of the ascending list a[0..na) that also occurs in the
// ascending list b[0..nb): out[0] = its index in a (na if none), out[1] = its
// index in b (-1 if none).  One CTA; every element of a is binary-searched in b
// in parallel and the smallest hit index wins.
__global__ void __launch_bounds__(1024) k_first_common(const int64_t *a, uint64_t na, const int64_t *b, uint64_t nb,
                                                       int64_t *out) {
    __shared__ unsigned long long best;  // (index in a << 32) | index in b
    if (threadIdx.x == 0) best = ~0ull;
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < na; i += blockDim.x) {
        const int64_t x = a[i];
        uint64_t lo = 0, hi = nb;  // first b[k] >= x
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (b[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        if (lo < nb && b[lo] == x) atomicMin(&best, ((unsigned long long)i << 32) | (unsigned long long)lo);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (best == ~0ull) {
            out[0] = (int64_t)na;
            out[1] = -1;
        } else {
            out[0] = (int64_t)(best >> 32);
            out[1] = (int64_t)(best & 0xFFFFFFFFull);
        }
    }
}

// ------------------------------------------------------------------ primitives (§4.1, §4.2)
// One warp per region.  The region is walked in 512-byte warp blocks of
// 16-byte aligned lane vectors; bytes outside the region are masked.
template <bool MAX>
__global__ void k_ebs(const uint8_t *data, const uint64_t *off, const uint64_t *len, uint64_t n, uint8_t *value,
                      uint64_t *pos) {
    const uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    if (r >= n) return;
    const uint8_t *b = data + off[r];
    const uint8_t *a0 = reinterpret_cast<const uint8_t *>(reinterpret_cast<uintptr_t>(b) & ~(uintptr_t)15);
    const int64_t lo = b - a0, hi = lo + (int64_t)len[r];  // region = [lo, hi) relative to a0
    // tree leaves: per-lane extreme; root: warp reduction
    uint32_t acc = neutral<MAX>();
    for (int64_t B = 0; B < hi; B += BLK) {
        const int rlo = lo - B > 0 ? (int)(lo - B) : 0, rhi = hi - B < BLK ? (int)(hi - B) : BLK;
        int la, lb;
        lane_part(rlo, rhi, la, lb);
        if (la < lb) {
            Blk k;
            k.v = *reinterpret_cast<const uint4 *>(a0 + B + lane * 16);
            acc = ext2<MAX>(acc, vext16_range<MAX>(k.v, la, lb));
        }
    }
    const uint32_t m = warp_ext<MAX>(acc);
    // leftmost occurrence: Range Scan with EQ
    for (int64_t B = 0; B < hi; B += BLK) {
        const int rlo = lo - B > 0 ? (int)(lo - B) : 0, rhi = hi - B < BLK ? (int)(hi - B) : BLK;
        int la, lb;
        lane_part(rlo, rhi, la, lb);
        Blk k;
        k.v = make_uint4(0, 0, 0, 0);
        uint32_t le = neutral<MAX>();
        if (la < lb) {
            k.v = *reinterpret_cast<const uint4 *>(a0 + B + lane * 16);
            le = vext16_range<MAX>(k.v, la, lb);
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, la < lb && le == m);
        if (bal) {
            const int q = locate<CMP_EQ>(k, bal, rlo, rhi, m);
            if (lane == 0) {
                value[r] = (uint8_t)m;
                pos[r] = (uint64_t)(B + q - lo);
            }
            return;
        }
    }
}

template <int CMP>
__global__ void k_range_scan(const uint8_t *data, const uint64_t *off, const uint64_t *len, const uint8_t *target,
                             uint64_t n, uint64_t *pos) {
    const uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    if (r >= n) return;
    const uint8_t *b = data + off[r];
    const uint64_t L = len[r];
    const uint32_t t = target[r];
    const uint8_t *a0 = reinterpret_cast<const uint8_t *>(reinterpret_cast<uintptr_t>(b) & ~(uintptr_t)15);
    const int64_t lo = b - a0, hi = lo + (int64_t)L;
    for (int64_t B = 0; B < hi; B += BLK) {
        const int rlo = lo - B > 0 ? (int)(lo - B) : 0, rhi = hi - B < BLK ? (int)(hi - B) : BLK;
        int la, lb;
        lane_part(rlo, rhi, la, lb);
        Blk k;
        k.v = make_uint4(0, 0, 0, 0);
        bool any = false;
        if (la < lb) {
            k.v = *reinterpret_cast<const uint4 *>(a0 + B + lane * 16);
            // packed scan of the lane's bytes (VCMP + VMASK, §4.2)
            for (int j = la; j < lb; ++j) any |= cmp_holds<CMP>(vbyte(k.v, j), t);
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, any);
        if (bal) {
            const int q = locate<CMP>(k, bal, rlo, rhi, t);
            if (lane == 0) pos[r] = (uint64_t)(B + q - lo);
            return;
        }
    }
    if (lane == 0) pos[r] = L;
}

}  // namespace cdc

// ====================================================================== host side
namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

// Optional per-kernel timing (cdc_profile_*): CUDA events recorded on the
// launching stream around each pipeline kernel of cdc_chunk / cdc_chunk_batch.
constexpr int PROF_KERNELS = 3;  // k_seg_prefix, k_speculate, k_fixup
struct ProfCall {
    cudaEvent_t ev[PROF_KERNELS + 1];
    bool used[PROF_KERNELS];
};
thread_local bool g_prof_on = false;
thread_local std::vector<ProfCall> g_prof_calls;
thread_local std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
    cudaEvent_t e;
    if (!g_prof_pool.empty()) {
        e = g_prof_pool.back();
        g_prof_pool.pop_back();
    } else {
        cudaEventCreate(&e);
    }
    return e;
}

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char *where) {
    return fail(CDC_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CDC_CUDA(call)                                   \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

// CDC_SYNC_DEBUG=1 in the environment: synchronise after every kernel and name
// the one that failed (debugging aid; never set in measurements).
bool sync_debug() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CDC_SYNC_DEBUG");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}
#define CDC_KCHECK(name, st)                                                   \
    do {                                                                       \
        if (sync_debug()) {                                                    \
            cudaError_t _e = cudaStreamSynchronize(st);                        \
            if (_e == cudaSuccess) _e = cudaGetLastError();                    \
            if (_e != cudaSuccess) return cuda_fail(_e, name);                 \
        }                                                                      \
    } while (0)

// Transfer tables are tried only for segments up to T_MAX_SEG: larger segments
// amortise their halos anyway, and a failed attempt (a stream saturated only
// in parts, such as configs[2]'s uniform base with zero-filled regions at
// 453 KB segments) costs ~5 % there.
#ifndef CDC_T_MAX_SEG
#define CDC_T_MAX_SEG (256ull << 10)
#endif
constexpr uint64_t T_MAX_SEG = CDC_T_MAX_SEG;

// Sparse walk (sparse_chain) for windows of at least SPARSE_MIN_W bytes: with
// shorter windows a chunk is little longer than the region a sparse step
// loads, and the streaming ring walker is faster.  CDC_SPARSE=0 disables it
// (a debugging and A/B knob).
#ifndef CDC_SPARSE_MIN_W
#define CDC_SPARSE_MIN_W 4096
#endif
constexpr uint32_t SPARSE_MIN_W = CDC_SPARSE_MIN_W;
int sparse_on(uint32_t w, uint64_t max_size) {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CDC_SPARSE");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    (void)max_size;
    return v && w >= SPARSE_MIN_W ? 1 : 0;
}

// CDC_TMODE=0 disables the transfer-table attempt (a debugging and testing knob)
int tmode_on() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CDC_TMODE");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v;
}

// CDC_FUSED=0 disables the fused look-back fast path (k_fixup always resolves;
// a debugging and testing knob)
int fused_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CDC_FUSED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v;
}

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor in the stream finishes; it calls griddepcontrol.wait
// before reading the predecessor's results.
template <typename... Args>
cudaError_t launch_pdl(const void *fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *pargs[] = {reinterpret_cast<void *>(&args)...};
    return cudaLaunchKernelExC(&cfg, fn, pargs);
}

int check_params(const cdc_params *p) {
    if (!p) return fail(CDC_ERR_INVALID, "null params");
    if (p->algo < CDC_RAM || p->algo > CDC_MAXP) return fail(CDC_ERR_INVALID, "unknown algorithm");
    if (p->window < 1) return fail(CDC_ERR_INVALID, "window must be >= 1");
    if (p->algo == CDC_MAXP && p->window > cdc::MX_HMAX)
        return fail(CDC_ERR_INVALID, "MAXP window must be <= 65536 (a tile's shared memory holds both windows)");
    // device code keeps w + 1 in 32-bit signed arithmetic
    if (p->window >= (1u << 31)) return fail(CDC_ERR_INVALID, "window must be < 2^31");
    if (p->max_size <= p->window) return fail(CDC_ERR_INVALID, "max_size must exceed window");
    if (p->seg_bytes % 16) return fail(CDC_ERR_INVALID, "seg_bytes must be a multiple of 16");
    if (p->seg_bytes && p->seg_bytes >= (1ull << 31)) return fail(CDC_ERR_INVALID, "seg_bytes too large");
    if (p->halo_bytes >= (1ull << 31)) return fail(CDC_ERR_INVALID, "halo_bytes too large");
    return CDC_OK;
}

// Per-device host state: the SM count and whether the kernels' dynamic shared
// memory opt-in (a per-device function attribute) has been set on the device.
constexpr int MAX_DEVICES = 64;
#define CDC_HOST_GROUPS_MAX 8
constexpr uint64_t CDC_HOST_GROUP_BYTES = 1ull << 30;  // cdc_chunk_batch_host: pipeline group size
int g_num_sms[MAX_DEVICES] = {0};
int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return (dev >= 0 && dev < MAX_DEVICES) ? dev : 0;
}
int num_sms() {
    const int dev = current_device();
    if (!g_num_sms[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        g_num_sms[dev] = n > 0 ? n : 148;
    }
    return g_num_sms[dev];
}

struct Plan {
    uint64_t S, Hmax, max_segs, cap_list, cap_halo, pool_cap, exc_cap, nfiles, poolb_cap;
    size_t bytes, reset_bytes;
    size_t off[40];
    // K-phase speculation (cdc_kphase.cuh): kK chains per segment (0 = off)
    uint32_t kK, kG, kD, kcap;
    uint64_t kS, kHk;
    size_t koff[4], kreset_bytes;
    // dense-index mode (cdc_dense.cuh): dG segments of dS bytes (0 = off)
    uint32_t dG, dS, dsteps, dext;
    size_t doff[6];
};

// cdc_set_dense / CDC_DENSE in the environment: 0 disables the dense-index mode
std::atomic<int> g_dense{-2};  // (-2: not read from the environment yet)
bool dense_on() {
    int v = g_dense.load();
    if (v == -2) {
        const char *e = getenv("CDC_DENSE");
        v = e ? atoi(e) : -1;
        int expect = -2;
        g_dense.compare_exchange_strong(expect, v);
        v = g_dense.load();
    }
    return v != 0;
}

// CDC_KPHASE in the environment: 0 disables K-phase speculation, 1..8 forces
// that many chains per segment; by default 4 for RAM with windows of 12 KiB and
// more (RAM at 16 KiB), else 2 (measured on configs[2]'s 1 GiB base, DESIGN.md
// §6).  AE with such windows also takes 4 below 512 MiB: on a stream without
// zero-filled regions two chains half a chunk apart meet only after ~(w / 2 /
// 362)^2 = 500 chunks (uniform 256 MiB, AE-Max 16 KiB: 0.90 ms with K = 2, 0.29 ms
// with 4), while configs[2]'s 1 GiB streams, whose zero-filled regions bring AE
// chains together, run 15 % faster with 2 (0.38 against 0.45 ms).  CDC_KSEGS
// overrides its segment count.
std::atomic<int> g_kphase{-2};  // cdc_set_kphase (-2: not read from the environment yet)
int kphase_k(int algo, uint32_t w, uint64_t total_len) {
    int v = g_kphase.load();
    if (v == -2) {
        const char *e = getenv("CDC_KPHASE");
        v = e ? atoi(e) : -1;
        int expect = -2;
        g_kphase.compare_exchange_strong(expect, v);
        v = g_kphase.load();
    }
    if (v == 0) return 0;
    if (v > 0) return std::min(v, cdc::KP_MAXK);
    return (w >= 12288 && (algo == CDC_RAM || total_len <= (512ull << 20))) ? 4 : 2;
}
uint64_t kphase_segs() {
    static long long v = -2;
    if (v == -2) {
        const char *e = getenv("CDC_KSEGS");
        v = e ? atoll(e) : 0;
    }
    return v > 0 ? (uint64_t)v : 0;
}

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Segment size: about SEGS_PER_SM walkers per SM for the total input (so the
// grid is a whole number of waves of SPEC_WARPS-warp CTAs), a multiple of the
// TMA stage, at least 64 KiB and 4 max-size chunks, so that the
// re-synchronisation halo (a few chunks on typical data) is small next to it.
constexpr uint64_t SEGS_PER_SM = (uint64_t)cdc::SPEC_WARPS * cdc::SPEC_CTAS_PER_SM;
constexpr uint64_t BATCH_SEGS_PER_SM = (uint64_t)cdc::BATCH_WARPS * cdc::SPEC_CTAS_PER_SM;
constexpr uint64_t FIX_BLOCKS = 16;  // k_fixup grid cap

void make_plan(const cdc_params *p, uint64_t nfiles, uint64_t total_len, uint64_t max_len, Plan &P) {
    uint64_t S = p->seg_bytes;
    if (!S) {
        const uint64_t target = (uint64_t)num_sms() * (nfiles > 1 ? BATCH_SEGS_PER_SM : SEGS_PER_SM);
        // floor(len / target): floor(len / S) = target segments of ~equal length
        S = total_len / target;
        // a batch: segments are taken largest first (LptLists), so only a file
        // longer than every other walker's share sets the tail -- cut such files
        // into segments shorter than one walker's share (a file's segments are
        // [S, 2S) long).  Long windows keep whole-share segments: their halos
        // re-synchronise slowly on saturated bytes.
        if (nfiles > 1 && p->window <= 8192) S /= 2;
        const uint64_t lo = std::max<uint64_t>(64 << 10, round_up(4 * p->max_size, 128));
        if (S < lo) S = lo;
        if (S > (256ull << 20)) S = 256ull << 20;
    }
    // halo cap: chains started at arbitrary offsets meet within a few chunks on
    // skewed data but only after ~(w/362)^2 chunks on uniform bytes (the phase
    // difference of two chains random-walks): 1024 windows, <= 64 MiB
    // (batches of many small files keep 64 windows: their segments are mostly whole
    // files, and the fix-up walkers continue any halo that gives up)
    const uint64_t hw = nfiles > 1 ? 64ull : 1024ull;
    const uint64_t w1 = (uint64_t)p->window + 1;
    uint64_t H = p->halo_bytes ? p->halo_bytes
                               : std::min<uint64_t>(std::max<uint64_t>(2 * S, hw * w1), 64ull << 20);
    if (H >= (1ull << 31)) H = (1ull << 31) - 1;
    P.S = S;
    P.Hmax = H;
    P.nfiles = nfiles;
    P.max_segs = (nfiles <= 1) ? (max_len + S - 1) / S + 1 : total_len / S + nfiles + 1;
    // a segment holds less than 2S + 4096 + n bytes (n = segments of its file,
    // at most max_len / S): seg_start rounds starts down to 4 KiB, and
    // floor(len / n) < 2S.  Every chunk but a file's last is longer than w.
    P.cap_list = (2 * S + 4096 + max_len / S + 1) / w1 + 2;
    P.cap_halo = H / w1 + 3;
    P.pool_cap = P.max_segs * P.cap_halo;  // one slice of cap_halo entries per segment
    P.poolb_cap = total_len / w1 + 2;
    P.exc_cap = P.max_segs;
    const uint64_t G = P.max_segs;
    // lists: a single stream's segments share one capacity; a batch sizes each
    // segment's list by its length (k_seg_prefix), len / (w+1) + 2 entries
    const uint64_t list_entries = nfiles > 1 ? total_len / w1 + 2 * G + 2 : G * P.cap_list;
    size_t sz[] = {
        list_entries * 4,    // 0 list   } reset to 0xFF by k_reset at every call
        G * 20 + 72 + (G / 32 + 1) * 12,  // 1 pub, status, ctrl, fetched, grp, tblk, tnx }
        G * P.cap_halo * 4,  // 2 halo
        G * 4,               // 3 cnt
        G * 4,               // 4 hcnt
        G * 4,               // 5 sj
        G * 4,               // 6 sa
        G * 4,               // 7 sb
        G * 4,               // 8 entry
        G * 4,               // 9 tail
        G * 4,               // 10 wcnt
        G * 4,               // 11 jump_entry
        G * 8,               // 12 woff
        G,                   // 13 skipped
        (G + 1) * 8,         // 14 seg_out
        G * 4,               // 15 exc
        G * 8,               // 16 ranges
        P.pool_cap * 4,      // 17 pool
        (nfiles + 1) * 8,    // 18 seg_first
        (nfiles + 1) * 8,    // 19 file_out
        64,                  // 20 misc
        G * 4,               // 21 seg_file
        G * 4,               // 22 ocnt
        G * 8,               // 23 ooff
        P.poolb_cap * 8,     // 24 poolb
        G * cdc::TK * 4,     // 25 tl
        G * cdc::TK * 4,     // 26 tn
        G * 4,               // 27 tk
        G * cdc::TK * 4,     // 28 tp
        G * cdc::TK * 4,     // 29 tq
        (G / cdc::TB + 2) * cdc::TK * 4,  // 30 tbc
        (G / cdc::TB + 2) * cdc::TK * 4,  // 31 tbs
        (G / cdc::TB + 2) * 4,            // 32 tbe
        (G / cdc::TB + 2) * 8,            // 33 tbo
        G * cdc::TEX * 8,                 // 34 tex
        (G + 2) * 8,                      // 35 lofs (batch)
        (2 * (total_len >> cdc::LPT_MIN_LOG2) + cdc::LPT_CLASSES + 1) * 4,  // 36 lpt lists (batch)
    };
    size_t o = 0;
    for (int i = 0; i < 37; ++i) {
        P.off[i] = o;
        o += round_up(sz[i], 256);
    }
    P.reset_bytes = P.off[2];
    // K-phase speculation: a single stream whose window takes the sparse walk,
    // when the transfer tables are not tried (their segments are longer than
    // T_MAX_SEG) and the segments are short next to the distance at which
    // chains started at random offsets meet on saturated bytes (mean ~600 KB
    // at RAM 8 KiB, ~2 MB at 16 KiB: configs[2]); longer segments amortise
    // their halos (configs[4]'s 8 GiB per GPU: 3.6 MB segments, where K
    // chains would only multiply the body walks).  Same segments as the
    // ordinary plan, K nodes each.
    // A small stream with default segments (the dense-index mode's range, below)
    // takes K-phase as well, behind the dense attempt and in front of the
    // transfer tables: the dense mode resolves what is saturated everywhere, and
    // on anything else (versioned data with zero-filled regions) a failed table
    // attempt leaves one speculative chain per segment, whose halos cost 2-20x
    // the K-phase walk (64 MiB versioned, RAM 16 KiB: 7.8 ms against 0.43 ms).
    // Such a stream has fewer nodes than walkers, so K is raised until they match.
    P.kK = 0;
    const bool small = nfiles <= 1 && dense_on() && p->seg_bytes == 0 && p->halo_bytes == 0 && p->window >= 4096 &&
                       p->window <= cdc::DN_WMAX && p->max_size >= 2ull * p->window + 2 &&
                       total_len >= (1ull << 20) && total_len <= (64ull << 20);
    int K = nfiles <= 1 ? kphase_k(p->algo, p->window, total_len) : 0;
    const bool tm = tmode_on() && p->window >= 4096 && S <= T_MAX_SEG;
    const uint64_t kmax_seg = kphase_segs() ? ~0ull : (p->window >= 12288 ? 4ull << 20 : 1ull << 20);
    // (default segments: K-phase also in front of the transfer tables' range -- a failed table attempt on a
    // stream saturated only in parts costs far more than the tables win on one saturated everywhere:
    // 128 MiB versioned, RAM 16 KiB, 10.7 ms against 0.48 ms)
    const bool prefer_k = p->seg_bytes == 0 && p->halo_bytes == 0 && dense_on();
    if (K > 0 && total_len > 0 && sparse_on(p->window, p->max_size) && (!tm || small || prefer_k) && S <= kmax_seg) {
        uint64_t Sk = S;
        if (kphase_segs()) Sk = std::max<uint64_t>(round_up(total_len / kphase_segs(), 4096), 64 << 10);
        uint64_t Gk = cdc::nseg_of(total_len, Sk);
        if ((small || prefer_k) && g_kphase.load() < 0 && Gk > 0)  // (the default K only: cdc_set_kphase / CDC_KPHASE force theirs)
            K = (int)std::min<uint64_t>(cdc::KP_MAXK, std::max<uint64_t>((uint64_t)K, (uint64_t)num_sms() * cdc::SPEC_WARPS / Gk));
        if (Gk * K > cdc::KNODE_MAX) {
            Sk = round_up(total_len / (cdc::KNODE_MAX / K) + 1, 4096);
            Gk = cdc::nseg_of(total_len, Sk);
        }
        const uint64_t Hk = p->halo_bytes ? p->halo_bytes : 1024 * w1;
        const uint64_t body = (2 * Sk + 4096 + Gk + 1) / w1 + 2;  // (the same bound as cap_list)
        const uint64_t capk = round_up(body + Hk / w1 + 4, 4);
        if (Gk >= 8 && Gk * K <= cdc::KNODE_MAX && capk < 65536) {
            const uint64_t N = Gk * K, NB = (Gk + cdc::KB - 1) / cdc::KB;
            P.kK = (uint32_t)K;
            P.kG = (uint32_t)Gk;
            P.kS = Sk;
            P.kHk = Hk;
            P.kcap = (uint32_t)capk;
            P.kD = std::max<uint32_t>(16u, ((p->window + 256u) / (uint32_t)K) & ~15u);
            size_t ksz[] = {
                N * capk * 4 + round_up(N * 4, 256) + 256,  // list, pub, ctrl } reset
                N * 4 * 4,                                  // nxt, idx, bxi, bval
                NB * 16,                                    // ent
                256,                                        // gate
            };
            for (int i = 0; i < 4; ++i) {
                P.koff[i] = o;
                o += round_up(ksz[i], 256);
            }
            P.kreset_bytes = round_up(ksz[0], 256);
        }
    }
    // Dense-index mode: a single stream of 1-64 MiB with the default segments,
    // a window the sparse walk would take and a cap no saturated chunk reaches.
    // Whether the stream is saturated everywhere is found out by the kernels;
    // the ordinary pipeline runs behind their gate otherwise.
    P.dG = 0;
    if (small) {
        const uint64_t nsm = (uint64_t)num_sms();
        const uint64_t Sd = std::min<uint64_t>(std::max<uint64_t>(round_up((total_len + nsm - 1) / nsm, 4096), cdc::DN_SMIN),
                                               cdc::DN_SMAX);
        const uint64_t Gd = total_len / Sd;
        if (Gd >= 2 && Gd <= (uint64_t)cdc::DN_GMAX) {
            P.dG = (uint32_t)Gd;
            P.dS = (uint32_t)Sd;
            P.dsteps = (uint32_t)(2 * Sd / w1 + 2);
            P.dext = 2 * p->window + 32;
            size_t dsz[] = {
                256,                                             // ctrl (reset)
                256,                                             // gate
                (Gd + 1) * 4,                                    // nc
                Gd * cdc::DN_CAND * 4,                           // tab
                Gd * cdc::DN_CAND * (size_t)P.dsteps * 4,        // rows
                Gd * 8,                                          // ent
            };
            for (int i = 0; i < 6; ++i) {
                P.doff[i] = o;
                o += round_up(dsz[i], 256);
            }
        }
    }
    P.bytes = o;
}

cdc::DGeo dgeo(const cdc_params *p, const Plan &P, const uint8_t *data, uint64_t len) {
    cdc::DGeo Q;
    Q.data = data;
    Q.L = len;
    Q.G = P.dG;
    Q.S = P.dS;
    Q.w = p->window;
    Q.steps = P.dsteps;
    Q.ext = P.dext;
    Q.ram = p->algo == CDC_RAM ? 1 : 0;
    Q.max = p->algo == CDC_AE_MIN ? 0 : 1;
    return Q;
}
cdc::DWork dcarve(const Plan &P, void *ws) {
    uint8_t *b = static_cast<uint8_t *>(ws);
    cdc::DWork X;
    X.ctrl = reinterpret_cast<unsigned long long *>(b + P.doff[0]);
    X.gate = reinterpret_cast<uint32_t *>(b + P.doff[1]);
    X.nc = reinterpret_cast<uint32_t *>(b + P.doff[2]);
    X.tab = reinterpret_cast<uint32_t *>(b + P.doff[3]);
    X.rows = reinterpret_cast<uint32_t *>(b + P.doff[4]);
    X.ent = reinterpret_cast<uint64_t *>(b + P.doff[5]);
    return X;
}

cdc::KGeo kgeo(const cdc_params *p, const Plan &P, const uint8_t *data, uint64_t len) {
    cdc::KGeo Q;
    Q.data = data;
    Q.L = len;
    Q.G = P.kG;
    Q.K = P.kK;
    Q.D = P.kD;
    Q.capk = P.kcap;
    Q.w = p->window;
    Q.max_size = p->max_size;
    Q.Hk = P.kHk;
    Q.sparse = sparse_on(p->window, p->max_size);
    Q.skip = nullptr;
    return Q;
}
cdc::KWork kcarve(const Plan &P, void *ws) {
    uint8_t *b = static_cast<uint8_t *>(ws);
    const uint64_t N = (uint64_t)P.kG * P.kK;
    cdc::KWork K;
    K.list = reinterpret_cast<uint32_t *>(b + P.koff[0]);
    K.pub = K.list + N * P.kcap;
    K.ctrl = reinterpret_cast<uint32_t *>(b + P.koff[0] + N * P.kcap * 4 + round_up(N * 4, 256));
    K.nxt = reinterpret_cast<uint32_t *>(b + P.koff[1]);
    K.idx = K.nxt + N;
    K.bxi = K.idx + N;
    K.bval = reinterpret_cast<int32_t *>(K.bxi + N);
    K.ent = reinterpret_cast<uint64_t *>(b + P.koff[2]);
    K.gate = reinterpret_cast<uint32_t *>(b + P.koff[3]);
    return K;
}

cdc::Work carve(const Plan &P, void *ws) {
    uint8_t *b = static_cast<uint8_t *>(ws);
    cdc::Work W;
    W.list = (uint32_t *)(b + P.off[0]);
    W.pub = (unsigned long long *)(b + P.off[1]);
    W.status = W.pub + P.max_segs;
    W.ctrl = reinterpret_cast<uint32_t *>(W.status + P.max_segs);
    W.fetched = W.status + P.max_segs + 8;
    W.grp = W.status + P.max_segs + 9;
    W.tblk = reinterpret_cast<uint32_t *>(W.grp + P.max_segs / 32 + 1);
    W.tnx = W.tblk + P.max_segs / 32 + 1;
    W.halo = (uint32_t *)(b + P.off[2]);
    W.cnt = (uint32_t *)(b + P.off[3]);
    W.hcnt = (uint32_t *)(b + P.off[4]);
    W.sj = (int32_t *)(b + P.off[5]);
    W.sa = (uint32_t *)(b + P.off[6]);
    W.sb = (uint32_t *)(b + P.off[7]);
    W.entry = (uint32_t *)(b + P.off[8]);
    W.tail = (uint32_t *)(b + P.off[9]);
    W.wcnt = (uint32_t *)(b + P.off[10]);
    W.jump_entry = (uint32_t *)(b + P.off[11]);
    W.woff = (uint64_t *)(b + P.off[12]);
    W.skipped = (uint8_t *)(b + P.off[13]);
    W.seg_out = (uint64_t *)(b + P.off[14]);
    W.exc = (uint32_t *)(b + P.off[15]);
    W.ranges = (uint32_t *)(b + P.off[16]);
    W.pool = (uint32_t *)(b + P.off[17]);
    W.seg_first = (uint64_t *)(b + P.off[18]);
    W.file_out = (uint64_t *)(b + P.off[19]);
    W.misc = (uint32_t *)(b + P.off[20]);
    W.seg_file = (uint32_t *)(b + P.off[21]);
    W.ocnt = (uint32_t *)(b + P.off[22]);
    W.ooff = (uint64_t *)(b + P.off[23]);
    W.poolb = (uint64_t *)(b + P.off[24]);
    W.tl = (uint32_t *)(b + P.off[25]);
    W.tn = (uint32_t *)(b + P.off[26]);
    W.tk = (uint32_t *)(b + P.off[27]);
    W.tp = (uint32_t *)(b + P.off[28]);
    W.tq = (uint32_t *)(b + P.off[29]);
    W.tbc = (uint32_t *)(b + P.off[30]);
    W.tbs = (uint32_t *)(b + P.off[31]);
    W.tbe = (uint32_t *)(b + P.off[32]);
    W.tbo = (uint64_t *)(b + P.off[33]);
    W.tex = (int64_t *)(b + P.off[34]);
    W.lofs = nullptr;  // set by run_chunk for batch calls (slots 35, 36)
    W.lpt = nullptr;
    W.poolb_cap = P.poolb_cap;
    W.cap_list = P.cap_list;
    W.cap_halo = P.cap_halo;
    W.pool_cap = P.pool_cap;
    W.max_segs = P.max_segs;
    W.exc_cap = P.exc_cap;
    return W;
}

template <int ALGO>
int launch_pipeline(const cdc_params *p, const Plan &P, cdc::Geometry &G, cdc::Work &W, uint64_t *d_bounds,
                    uint64_t cap, uint64_t *d_count, uint64_t *file_out, cudaStream_t st, bool batch,
                    uint64_t total_len) {
    static bool attr_set[MAX_DEVICES] = {false};  // per device: the opt-in is a per-context attribute
    const int spec_smem = cdc::SPEC_WARPS * cdc::RING_SMEM + 128;
    const int batch_smem = cdc::BATCH_WARPS * cdc::Ring<cdc::BATCH_STAGE>::SMEM + 128;
    const int dev = current_device();
    if (!attr_set[dev]) {
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_speculate<ALGO, false, cdc::BATCH_WARPS, cdc::BATCH_STAGE, false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, batch_smem));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_speculate<ALGO, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      spec_smem));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_speculate<ALGO, false, cdc::SPEC_WARPS, cdc::STAGE, true, 0>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, spec_smem));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_speculate<ALGO, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      spec_smem));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_fixup<ALGO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      cdc::FIX_SMEM));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_kspec<ALGO>, cudaFuncAttributeMaxDynamicSharedMemorySize, spec_smem));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_kres2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(cdc::KNODE_MAX * 8)));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_kres_all, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(cdc::KRES_ALL_NB * cdc::KB * cdc::KP_MAXK * 8)));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_dense_index, cudaFuncAttributeMaxDynamicSharedMemorySize, cdc::DN_SMEM));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_dense_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize, cdc::DN_SMEM));
        attr_set[dev] = true;
    }
    int launches = 0;
    ProfCall pc{};
    auto mark = [&](int i) {
        if (g_prof_on) {
            pc.ev[i] = prof_event();
            cudaEventRecord(pc.ev[i], st);
        }
    };
    mark(0);
    bool dense_reset = false;  // the reset below is part of k_dense_finish
    const uint32_t *dense_gate = nullptr;
    if (P.dG && !batch) {
        // dense-index mode (cdc_dense.cuh); the ordinary pipeline behind it runs
        // only if its gate opens (the stream is not saturated everywhere)
        const cdc::DGeo Q = dgeo(p, P, G.data, total_len);
        const cdc::DWork X = dcarve(P, W.list);
        cdc::k_dense_index<<<(unsigned)std::min<uint64_t>(Q.G, (uint64_t)num_sms()), cdc::DN_THREADS, cdc::DN_SMEM, st>>>(Q, X);
        CDC_KCHECK("k_dense_index", st);
        CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_dense_resolve), dim3(1), dim3(cdc::DN_THREADS),
                            (size_t)cdc::DN_SMEM, st, Q, X));
        CDC_KCHECK("k_dense_resolve", st);
        // (k_dense_finish writes the output, or is the list reset of what follows when the gate opened:
        // K-phase's lists, else the ordinary pipeline's)
        const uint64_t n16 = (P.kK ? P.kreset_bytes : P.reset_bytes) / 16;
        uint4 *rst = reinterpret_cast<uint4 *>(P.kK ? (void *)kcarve(P, W.list).list : (void *)W.list);
        const unsigned rb = (unsigned)std::min<uint64_t>((n16 + 255) / 256, 4 * (uint64_t)num_sms());
        CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_dense_finish), dim3(std::max(rb, (Q.G + 7) / 8)),
                            dim3(256), 0, st, Q, X, d_bounds, cap, d_count, rst, n16));
        CDC_KCHECK("k_dense_finish", st);
        launches += 3;
        G.gate = X.gate;
        G.gate0 = X.gate;
        dense_reset = true;
        dense_gate = X.gate;
    }
    if (P.kK) {
        // K-phase speculation (cdc_kphase.cuh); the ordinary pipeline behind it
        // runs only if its gate opens (a halo on the true chain gave up)
        cdc::KGeo Q = kgeo(p, P, G.data, total_len);
        Q.skip = dense_gate;  // (behind the dense-index mode: nothing to do when its gate stayed shut)
        const cdc::KWork KW = kcarve(P, W.list);
        const uint64_t N = (uint64_t)Q.G * Q.K, NB = (Q.G + cdc::KB - 1) / cdc::KB;
        if (!dense_reset) {
            const uint64_t n16 = P.kreset_bytes / 16;
            const unsigned rb = (unsigned)std::min<uint64_t>((n16 + 255) / 256, 4 * (uint64_t)num_sms());
            cdc::k_reset<<<rb ? rb : 1, 256, 0, st>>>(reinterpret_cast<uint4 *>(KW.list), n16, nullptr);
            CDC_KCHECK("k_reset (K-phase)", st);
            ++launches;
        }
        dense_reset = false;  // the ordinary pipeline's own (gated) reset follows
        CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_kspec<ALGO>),
                            dim3((unsigned)std::min<uint64_t>((N + cdc::SPEC_WARPS - 1) / cdc::SPEC_WARPS,
                                                              (uint64_t)num_sms())),
                            dim3(cdc::SPEC_WARPS * 32), (size_t)spec_smem, st, Q, KW));
        CDC_KCHECK("k_kspec", st);
        if (NB <= cdc::KRES_ALL_NB) {
            // a small stream: the three resolution levels in one CTA, which is also the
            // ordinary pipeline's list reset when a node on the true path gave up
            CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_kres_all), dim3(1), dim3(1024), (size_t)(N * 8),
                                st, Q, KW, d_count, d_bounds, cap, reinterpret_cast<uint4 *>(W.list),
                                (uint64_t)(P.reset_bytes / 16)));
            CDC_KCHECK("k_kres_all", st);
            launches += 2;
            dense_reset = true;  // (the ordinary pipeline's reset is part of k_kres_all)
        } else {
            CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_kres1),
                                dim3((unsigned)((NB + cdc::KRES1_WARPS - 1) / cdc::KRES1_WARPS)),
                                dim3(cdc::KRES1_WARPS * 32), 0, st, Q, KW));
            CDC_KCHECK("k_kres1", st);
            CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_kres2), dim3(1), dim3(1024), (size_t)(N * 8), st,
                                Q, KW, d_count));
            CDC_KCHECK("k_kres2", st);
            CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_kres3), dim3((unsigned)((NB + 7) / 8)), dim3(256),
                                0, st, Q, KW, d_bounds, cap));
            CDC_KCHECK("k_kres3", st);
            launches += 4;
        }
        G.gate = KW.gate;
    }
    // reset the published lists (list entries -> LIST_EMPTY, pub -> PUB_OPEN) and
    // the look-back, ticket and flag words
    if (!dense_reset) {
        const uint64_t n16 = P.reset_bytes / 16;  // reset_bytes is a multiple of 256
        const unsigned rb = (unsigned)std::min<uint64_t>((n16 + 255) / 256, 4 * (uint64_t)num_sms());
        if (G.gate)
            CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_reset), dim3(rb ? rb : 1), dim3(256), 0, st,
                                reinterpret_cast<uint4 *>(W.list), n16, G.gate, G.gate0));
        else
            cdc::k_reset<<<rb ? rb : 1, 256, 0, st>>>(reinterpret_cast<uint4 *>(W.list), n16, G.gate);
        CDC_KCHECK("k_reset", st);
        ++launches;
    }
    if (batch) {
        // segment table (launched with PDL behind the reset; k_speculate behind it)
        const uint64_t tiles = (G.nfiles + cdc::SP_THREADS * cdc::SP_RPT - 1) / (cdc::SP_THREADS * cdc::SP_RPT);
        const unsigned sb = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, 2 * (uint64_t)num_sms()));
        CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_seg_prefix), dim3(sb), dim3(cdc::SP_THREADS), 0,
                            st, G.file_off, G.nfiles, G.S, (uint64_t)p->window + 1, W.seg_first, W.seg_file,
                            W.lofs, W.status, W.ctrl + cdc::CT_SP_TICKET,
                            cdc::LptLists{W.tnx, W.tblk, W.lpt, total_len}));
        CDC_KCHECK("k_seg_prefix", st);
        ++launches;
        pc.used[0] = true;
    }
    mark(1);
    // segments: exact for a single stream (nseg_of), an upper bound for a batch
    const uint64_t nseg_ub = batch ? P.max_segs
                                   : (total_len == 0 ? 0 : (total_len < P.S ? 1 : total_len / P.S));
    // segments per CTA: SPEC_WARPS, or fewer when the input has fewer segments
    // than walkers fit on the GPU (one walker per SM for a small stream)
    const uint64_t nsm = (uint64_t)num_sms();
    // (a batch: spw = 0, one wave of CTAs whose warps take segments from a global
    // ticket, which balances files of very different sizes)
    const int spw = batch ? 0
                          : (int)std::min<uint64_t>(std::max<uint64_t>((nseg_ub + nsm - 1) / nsm, 1), cdc::SPEC_WARPS);
    const uint64_t blocks = batch ? std::min<uint64_t>((nseg_ub + cdc::BATCH_WARPS - 1) / cdc::BATCH_WARPS,
                                                       nsm * cdc::SPEC_CTAS_PER_SM)
                                  : (nseg_ub + spw - 1) / spw;
    // transfer tables: a single stream of at least two segments, windows long
    // enough for slow convergence, segments short enough for their halos to
    // matter, and a grid that is one co-resident wave (the attempt waits for
    // every walker; it also gives up after a timeout)
    G.tmode = (!batch && tmode_on() && p->window >= 4096 && P.S <= T_MAX_SEG && nseg_ub >= 3 &&
               blocks <= nsm) ? 1 : 0;
    if (blocks > 0) {
        // the fused look-back makes each segment wait for its predecessors: with
        // dynamic tickets (a batch) the waits would queue behind the largest file,
        // so a batch leaves the splice and the writes to k_fixup
        int fused = (!batch && P.cap_list + P.cap_halo < (1u << 23)) ? fused_mode() : 0;
        const void *kspec =
            batch ? reinterpret_cast<const void *>(cdc::k_speculate<ALGO, false, cdc::BATCH_WARPS, cdc::BATCH_STAGE, false>)
            : G.tmode ? reinterpret_cast<const void *>(cdc::k_speculate<ALGO, true>)
            : G.sparse ? reinterpret_cast<const void *>(cdc::k_speculate<ALGO, false>)
                       : reinterpret_cast<const void *>(cdc::k_speculate<ALGO, false, cdc::SPEC_WARPS, cdc::STAGE, true, 0>);
        CDC_CUDA(launch_pdl(kspec, dim3((unsigned)blocks), dim3((batch ? cdc::BATCH_WARPS : cdc::SPEC_WARPS) * 32),
                            (size_t)(batch ? batch_smem : spec_smem), st, G, W, d_bounds, cap, d_count, fused, spw));
        CDC_KCHECK("k_speculate", st);
        ++launches;
        pc.used[1] = true;
    }
    mark(2);
    {
        // a small grid: it exits at once in the common case; writers stride over segments otherwise
        // (a batch: the writers of every segment's boundaries span the GPU, two CTAs per SM)
        const uint64_t fblocks = std::min<uint64_t>((nseg_ub + 31) / 32, batch ? 2 * nsm : FIX_BLOCKS);
        CDC_CUDA(launch_pdl(reinterpret_cast<const void *>(cdc::k_fixup<ALGO>), dim3((unsigned)(fblocks ? fblocks : 1)),
                            dim3(cdc::RESOLVE_THREADS), (size_t)cdc::FIX_SMEM, st, G, W, d_count, file_out, d_bounds,
                            cap));
        CDC_KCHECK("k_fixup", st);
        ++launches;
        pc.used[2] = true;
    }
    mark(3);
    if (g_prof_on) g_prof_calls.push_back(pc);
    g_launches = launches;
    CDC_CUDA(cudaGetLastError());
    return CDC_OK;
}

// ------------------------------------------------------------------ MAXP (cdc_maxp.cuh)
struct MaxpPlan {
    cdc::MaxpGeo Q;
    uint64_t nlt;           // link / write tiles
    uint64_t ngc;           // k_maxp_gather CTAs
    uint64_t nfc;           // k_maxp_files CTAs
    size_t off_tfirst, off_tfile, off_qt, off_qn, off_qx, off_efile, off_estart, off_f, off_ncap, off_jl;
    size_t off_reset, reset_bytes, bytes;
    uint32_t smem;          // k_maxp_scan dynamic shared memory
};
uint32_t maxp_smem(uint64_t h, uint32_t &buf, uint32_t &ccap) {
    buf = (uint32_t)round_up(cdc::MX_TILE + 2 * h + 32, 128);
    ccap = (uint32_t)(cdc::MX_TILE / (h + 1) + 2);
    const uint32_t ng = buf / 16, nb = ng / cdc::MX_BG + 1;  // granule maxima, block maxima, survivors, candidates
    return buf + ng + ((nb + 1) & ~1u) + 2 * (ng / 2 + 1) + 2 * ccap + 128;
}
// nfiles streams totalling total bytes (a single stream: nfiles = 1)
void maxp_plan(const cdc_params *p, uint64_t nfiles, uint64_t total, MaxpPlan &P) {
    cdc::MaxpGeo &Q = P.Q;
    Q.data = nullptr;
    Q.file_off = nullptr;
    Q.nfiles = nfiles;
    Q.L = total;
    Q.h = p->window;
    Q.M = p->max_size;
    Q.ntiles = total / cdc::MX_TILE + nfiles;           // >= sum of max(1, ceil(len / MX_TILE))
    Q.qcap = total / (Q.h + 1) + 2 * nfiles + 2;         // maxima are > h apart; one start per file
    P.smem = maxp_smem(Q.h, Q.buf, Q.ccap);
    P.nlt = (Q.qcap + cdc::MX_ETILE - 1) / cdc::MX_ETILE;
    P.ngc = (Q.ntiles + cdc::MX_GTILES - 1) / cdc::MX_GTILES;
    P.nfc = (nfiles + cdc::MX_FTHREADS - 1) / cdc::MX_FTHREADS;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = round_up(o + bytes, 256);
        return at;
    };
    P.off_tfirst = take((nfiles + 1) * 8);
    P.off_tfile = take(Q.ntiles * 4);
    P.off_qt = take(Q.ntiles * Q.ccap * 2);
    P.off_qn = take(Q.ntiles * 4);
    P.off_qx = take(Q.qcap * 8);
    P.off_efile = take(Q.qcap * 4);
    P.off_estart = take((nfiles + 1) * 8);
    P.off_f = take(Q.qcap * 8);
    P.off_ncap = take(Q.qcap * 8);
    P.off_jl = take(Q.qcap * 8);
    P.off_reset = o;  // fst, tst, lst, wst, ctrl, nq, nj, on -- reset to all-ones by k_reset
    P.reset_bytes = round_up((P.nfc + P.ngc + 2 * P.nlt) * 8 + 32 + 16 + Q.qcap, 256);
    P.bytes = o + P.reset_bytes;
}
cdc::MaxpWork maxp_carve(const MaxpPlan &P, void *ws) {
    uint8_t *b = static_cast<uint8_t *>(ws);
    cdc::MaxpWork X;
    X.tfirst = reinterpret_cast<uint64_t *>(b + P.off_tfirst);
    X.tfile = reinterpret_cast<uint32_t *>(b + P.off_tfile);
    X.qt = reinterpret_cast<uint16_t *>(b + P.off_qt);
    X.qn = reinterpret_cast<uint32_t *>(b + P.off_qn);
    X.qx = reinterpret_cast<int64_t *>(b + P.off_qx);
    X.efile = reinterpret_cast<uint32_t *>(b + P.off_efile);
    X.estart = reinterpret_cast<uint64_t *>(b + P.off_estart);
    X.f = reinterpret_cast<int64_t *>(b + P.off_f);
    X.ncap = reinterpret_cast<uint64_t *>(b + P.off_ncap);
    X.jl = reinterpret_cast<int64_t *>(b + P.off_jl);
    X.bo = nullptr;
    unsigned long long *r = reinterpret_cast<unsigned long long *>(b + P.off_reset);
    X.fst = r;
    X.tst = X.fst + P.nfc;
    X.lst = X.tst + P.ngc;
    X.wst = X.lst + P.nlt;
    X.ctrl = reinterpret_cast<uint32_t *>(X.wst + P.nlt);
    X.nq = reinterpret_cast<unsigned long long *>(X.ctrl + 8);
    X.nj = X.nq + 1;
    X.on = reinterpret_cast<uint8_t *>(X.nj + 1);
    return X;
}

// MAXP over one stream (d_file_off null, nfiles 1) or a packed batch (d_bound_off
// receives each file's first output index).
int launch_maxp(const cdc_params *p, const uint8_t *d_data, const uint64_t *d_file_off, uint64_t nfiles,
                uint64_t total, uint64_t *d_bounds, uint64_t cap, uint64_t *d_bound_off, uint64_t *d_count, void *ws,
                size_t ws_bytes, cudaStream_t st) {
    MaxpPlan P;
    maxp_plan(p, nfiles, total, P);
    if (ws_bytes < P.bytes) return fail(CDC_ERR_WORKSPACE, "workspace too small");
    P.Q.data = d_data;
    P.Q.file_off = d_file_off;
    cdc::MaxpWork X = maxp_carve(P, ws);
    X.bo = d_bound_off;
    static bool attr[MAX_DEVICES] = {false};
    const int dev = current_device();
    if (!attr[dev]) {  // the largest window's tile (per device: a context attribute)
        uint32_t b, c;
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_maxp_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)maxp_smem(cdc::MX_HMAX, b, c)));  // (<= 227 KB: static_assert below)
        attr[dev] = true;
    }
    const uint64_t nsm = (uint64_t)num_sms();
    const uint64_t n16 = P.reset_bytes / 16;
    cdc::k_reset<<<(unsigned)std::min<uint64_t>((n16 + 255) / 256, 4 * nsm), 256, 0, st>>>(
        reinterpret_cast<uint4 *>(static_cast<uint8_t *>(ws) + P.off_reset), n16, nullptr);
    CDC_CUDA(cudaGetLastError());  // a launch error stops the pipeline here
    CDC_KCHECK("k_reset (MAXP)", st);
    cdc::k_maxp_files<<<(unsigned)P.nfc, cdc::MX_FTHREADS, 0, st>>>(P.Q, X);
    CDC_CUDA(cudaGetLastError());
    CDC_KCHECK("k_maxp_files", st);
    int per_sm = 0;
    CDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cdc::k_maxp_scan, cdc::MX_THREADS, P.smem));
    const uint64_t sblocks = std::min<uint64_t>(P.Q.ntiles, nsm * (uint64_t)std::max(per_sm, 1));
    cdc::k_maxp_scan<<<(unsigned)sblocks, cdc::MX_THREADS, P.smem, st>>>(P.Q, X);
    CDC_CUDA(cudaGetLastError());
    CDC_KCHECK("k_maxp_scan", st);
    cdc::k_maxp_gather<<<(unsigned)P.ngc, cdc::MX_GTILES, 0, st>>>(P.Q, X);
    CDC_CUDA(cudaGetLastError());
    CDC_KCHECK("k_maxp_gather", st);
    // element tiles: CTAs take them from a ticket (the grid covers the capacity; CTAs past the count exit)
    const unsigned eblocks = (unsigned)std::min<uint64_t>(P.nlt, 16 * nsm);
    cdc::k_maxp_link<<<eblocks, cdc::MX_ETILE, 0, st>>>(P.Q, X);
    CDC_CUDA(cudaGetLastError());
    CDC_KCHECK("k_maxp_link", st);
    cdc::k_maxp_path<<<1, 256, 0, st>>>(P.Q, X);
    CDC_CUDA(cudaGetLastError());
    CDC_KCHECK("k_maxp_path", st);
    cdc::k_maxp_write<<<eblocks, cdc::MX_ETILE, 0, st>>>(P.Q, X, d_bounds, cap, d_count);
    CDC_CUDA(cudaGetLastError());
    CDC_KCHECK("k_maxp_write", st);
    g_launches = 7;
    return CDC_OK;
}

int run_chunk(const cdc_params *p, const uint8_t *d_data, const uint64_t *d_file_off, uint64_t nfiles,
              uint64_t total_len, uint64_t max_len, uint64_t *d_bounds, uint64_t cap, uint64_t *d_bound_off,
              uint64_t *d_count, void *ws, size_t ws_bytes, void *stream, bool batch) {
    int rc = check_params(p);
    if (rc) return rc;
    if (!d_count || (!d_bounds && cap) || (total_len && !d_data) || !ws)
        return fail(CDC_ERR_INVALID, "null pointer argument");
    if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(CDC_ERR_INVALID, "workspace must be 256-byte aligned");
    if (p->algo == CDC_MAXP)
        return launch_maxp(p, d_data, batch ? d_file_off : nullptr, batch ? nfiles : 1, total_len, d_bounds, cap,
                           batch ? d_bound_off : nullptr, d_count, ws, ws_bytes, static_cast<cudaStream_t>(stream));
    Plan P;
    make_plan(p, nfiles, total_len, max_len, P);
    if (ws_bytes < P.bytes) return fail(CDC_ERR_WORKSPACE, "workspace too small");
    cdc::Work W = carve(P, ws);
    // a batch's lists are sized per segment (k_seg_prefix); for nfiles == 1 the
    // single-stream list region (G x cap_list) holds them as well
    if (batch) {
        W.lofs = reinterpret_cast<uint64_t *>(static_cast<uint8_t *>(ws) + P.off[35]);
        W.lpt = reinterpret_cast<uint32_t *>(static_cast<uint8_t *>(ws) + P.off[36]);
    }
    cdc::Geometry G;
    G.data = d_data;
    G.file_off = batch ? d_file_off : nullptr;
    G.L = batch ? 0 : total_len;
    G.total = total_len;
    G.nfiles = batch ? nfiles : 1;
    G.S = P.S;
    G.Hmax = P.Hmax;
    G.w = p->window;
    G.max_size = p->max_size;
    G.tmode = 0;
    G.sparse = sparse_on(p->window, p->max_size);
    G.gate = nullptr;
    G.gate0 = nullptr;
    uint64_t *file_out = batch ? d_bound_off : W.file_out;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (p->algo) {
    case CDC_RAM: return launch_pipeline<cdc::ALGO_RAM>(p, P, G, W, d_bounds, cap, d_count, file_out, st, batch, total_len);
    case CDC_AE_MAX: return launch_pipeline<cdc::ALGO_AE_MAX>(p, P, G, W, d_bounds, cap, d_count, file_out, st, batch, total_len);
    default: return launch_pipeline<cdc::ALGO_AE_MIN>(p, P, G, W, d_bounds, cap, d_count, file_out, st, batch, total_len);
    }
}

// cached device buffers for cdc_chunk_host / cdc_chunk_batch_host, one set per
// device and calling thread (kept until the thread exits)
struct HostCache {
    uint8_t *data = nullptr;
    size_t data_cap = 0;
    uint64_t *bounds = nullptr;
    size_t bounds_cap = 0;
    void *ws = nullptr;
    size_t ws_cap = 0;
    uint64_t *count = nullptr;      // [0] count, then per-group counts (batch)
    uint64_t *offs = nullptr;       // batch: rebased file offsets of every group
    size_t offs_cap = 0;
    uint64_t *bo = nullptr;         // batch: per-group bound offsets
    size_t bo_cap = 0;
    cudaStream_t st = nullptr;      // compute
    cudaStream_t cp = nullptr;      // host-to-device copies (batch pipeline)
    cudaEvent_t ev[CDC_HOST_GROUPS_MAX];
    bool init = false;
};
thread_local HostCache g_hc[MAX_DEVICES];

int host_cache(HostCache *&C) {
    const int dev = current_device();
    C = &g_hc[dev];
    if (!C->init) {
        CDC_CUDA(cudaStreamCreateWithFlags(&C->st, cudaStreamNonBlocking));
        CDC_CUDA(cudaStreamCreateWithFlags(&C->cp, cudaStreamNonBlocking));
        for (int i = 0; i < CDC_HOST_GROUPS_MAX; ++i) CDC_CUDA(cudaEventCreateWithFlags(&C->ev[i], cudaEventDisableTiming));
        CDC_CUDA(cudaMalloc(&C->count, 8 * (CDC_HOST_GROUPS_MAX + 1)));
        C->init = true;
    }
    return CDC_OK;
}

int ensure(void **p, size_t &cap, size_t need) {
    if (cap >= need && *p) return CDC_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    cap = 0;
    CDC_CUDA(cudaMalloc(p, need ? need : 16));
    cap = need;
    return CDC_OK;
}

}  // namespace

extern "C" {

int cdc_abi_version(void) { return CDC_ABI_VERSION; }

const char *cdc_last_error(void) { return g_err.c_str(); }

int cdc_last_launch_count(void) { return g_launches; }

int cdc_set_dense(int on) {
    if (on < -1 || on > 1) return fail(CDC_ERR_INVALID, "on must be -1 (default), 0 (off) or 1 (on)");
    if (on == -1) {
        const char *e = getenv("CDC_DENSE");
        on = e ? atoi(e) : -1;
    }
    g_dense.store(on);
    return CDC_OK;
}

int cdc_set_kphase(int k) {
    if (k < -1 || k > cdc::KP_MAXK) return fail(CDC_ERR_INVALID, "k must be -1 (default), 0 (off) or 1..8");
    if (k == -1) {
        const char *e = getenv("CDC_KPHASE");
        k = e ? atoi(e) : -1;
    }
    g_kphase.store(k);
    return CDC_OK;
}

// diagnostic (CDC_EVTIME builds): read and reset the 16 cycle buckets
extern "C" int cdc_debug_evtime(unsigned long long *out) {
    CDC_CUDA(cudaMemcpyFromSymbol(out, cdc::g_evt, 16 * sizeof(unsigned long long)));
    unsigned long long z[16] = {0};
    CDC_CUDA(cudaMemcpyToSymbol(cdc::g_evt, z, sizeof(z)));
    return CDC_OK;
}

// diagnostic (CDC_COUNTERS builds): read and reset the 16 event counters
extern "C" int cdc_debug_counters(unsigned long long *out) {
    CDC_CUDA(cudaMemcpyFromSymbol(out, cdc::g_cnt, 16 * sizeof(unsigned long long)));
    unsigned long long z[16] = {0};
    CDC_CUDA(cudaMemcpyToSymbol(cdc::g_cnt, z, sizeof(z)));
    return CDC_OK;
}

// diagnostic (CDC_WAIT_PROBE builds): read and reset the summed stage-wait time
extern "C" int cdc_debug_wait_ns(unsigned long long *ns) {
    CDC_CUDA(cudaMemcpyFromSymbol(ns, cdc::g_wait_ns, sizeof(*ns)));
    unsigned long long z = 0;
    CDC_CUDA(cudaMemcpyToSymbol(cdc::g_wait_ns, &z, sizeof(z)));
    return CDC_OK;
}

int cdc_plan_info(const cdc_params *p, uint64_t nfiles, uint64_t total_len, uint64_t max_len, uint64_t *out) {
    int rc = check_params(p);
    if (rc) return rc;
    if (p->algo == CDC_MAXP) return fail(CDC_ERR_INVALID, "not defined for MAXP (no speculative segments)");
    if (!out) return fail(CDC_ERR_INVALID, "null out");
    Plan P;
    make_plan(p, nfiles ? nfiles : 1, total_len, max_len, P);
    out[0] = P.S;
    out[1] = P.Hmax;
    out[2] = max_len == 0 ? 0 : (max_len < P.S ? 1 : max_len / P.S);
    return CDC_OK;
}

int cdc_debug_timing(void *d_buf) {
    unsigned long long *p = static_cast<unsigned long long *>(d_buf);
    CDC_CUDA(cudaMemcpyToSymbol(cdc::g_timing, &p, sizeof(p)));
    return CDC_OK;
}

int cdc_fetched(const cdc_params *p, uint64_t nfiles, uint64_t total_len, uint64_t max_len, const void *d_workspace,
                uint64_t *out, void *stream) {
    int rc = check_params(p);
    if (rc) return rc;
    if (p->algo == CDC_MAXP) return fail(CDC_ERR_INVALID, "not defined for MAXP (no speculative segments)");
    if (!d_workspace || !out) return fail(CDC_ERR_INVALID, "null pointer");
    Plan P;
    make_plan(p, nfiles ? nfiles : 1, total_len, max_len, P);
    const cdc::Work W = carve(P, const_cast<void *>(d_workspace));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned long long v = 0;
    CDC_CUDA(cudaMemcpyAsync(&v, W.fetched, 8, cudaMemcpyDeviceToHost, st));
    CDC_CUDA(cudaStreamSynchronize(st));
    *out = (uint64_t)(v + 1ull);  // the reset leaves ~0
    return CDC_OK;
}

int cdc_stats(const cdc_params *p, uint64_t nfiles, uint64_t total_len, uint64_t max_len, const void *d_workspace,
              uint64_t *stats, void *stream) {
    int rc = check_params(p);
    if (rc) return rc;
    if (p->algo == CDC_MAXP) return fail(CDC_ERR_INVALID, "not defined for MAXP (no speculative segments)");
    if (!d_workspace || !stats) return fail(CDC_ERR_INVALID, "null pointer");
    Plan P;
    make_plan(p, nfiles ? nfiles : 1, total_len, max_len, P);
    cdc::Work W = carve(P, const_cast<void *>(d_workspace));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (P.dG && nfiles <= 1) {  // dense-index mode, unless its gate sent the call to the ordinary pipeline
        const cdc::DWork X = dcarve(P, const_cast<void *>(d_workspace));
        uint32_t gate = 1;
        CDC_CUDA(cudaMemcpyAsync(&gate, X.gate, 4, cudaMemcpyDeviceToHost, st));
        CDC_CUDA(cudaStreamSynchronize(st));
        if (gate == 0) {
            stats[0] = P.dG;
            stats[1] = P.dS;
            stats[2] = P.dext;
            stats[3] = 4;  // resolved by the dense-index mode
            stats[4] = P.dG;
            stats[5] = stats[6] = stats[7] = 0;
            return CDC_OK;
        }
    }
    if (P.kK && nfiles <= 1) {  // K-phase: node statistics unless the gate sent the call to the ordinary pipeline
        const cdc::KWork KW = kcarve(P, const_cast<void *>(d_workspace));
        uint32_t gate = 1;
        CDC_CUDA(cudaMemcpyAsync(&gate, KW.gate, 4, cudaMemcpyDeviceToHost, st));
        CDC_CUDA(cudaStreamSynchronize(st));
        if (gate == 0) {
            const uint64_t N = (uint64_t)P.kG * P.kK;
            std::vector<uint32_t> nx(N), cn(N);
            CDC_CUDA(cudaMemcpyAsync(nx.data(), KW.nxt, N * 4, cudaMemcpyDeviceToHost, st));
            CDC_CUDA(cudaMemcpyAsync(cn.data(), KW.pub, N * 4, cudaMemcpyDeviceToHost, st));
            CDC_CUDA(cudaStreamSynchronize(st));
            uint64_t met = 0, uns = 0, other = 0, walked = 0;
            for (uint64_t v = 0; v < N; ++v) {
                if (nx[v] < cdc::KN_VOID) ++met;
                else if (nx[v] == cdc::KN_UNSYNC) ++uns;
                else ++other;
                walked += cn[v];
            }
            stats[0] = P.kG;
            stats[1] = P.kS;
            stats[2] = P.kHk;
            stats[3] = 3;  // resolved by K-phase speculation (stats[4..6] count nodes)
            stats[4] = met;
            stats[5] = uns;
            stats[6] = other;
            stats[7] = walked;
            return CDC_OK;
        }
    }
    uint64_t G = 0;
    if (nfiles <= 1 && P.S) G = max_len == 0 ? 0 : (max_len < P.S ? 1 : max_len / P.S);
    if (nfiles > 1) CDC_CUDA(cudaMemcpyAsync(&G, W.seg_first + nfiles, 8, cudaMemcpyDeviceToHost, st));
    uint32_t ctrl[2] = {0, 0};
    CDC_CUDA(cudaMemcpyAsync(ctrl, W.ctrl, 8, cudaMemcpyDeviceToHost, st));
    CDC_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> sj(G);
    std::vector<uint32_t> hc(G);
    if (G) {
        CDC_CUDA(cudaMemcpyAsync(sj.data(), W.sj, G * 4, cudaMemcpyDeviceToHost, st));
        CDC_CUDA(cudaMemcpyAsync(hc.data(), W.hcnt, G * 4, cudaMemcpyDeviceToHost, st));
        CDC_CUDA(cudaStreamSynchronize(st));
    }
    uint64_t met = 0, unsynced = 0, other = 0, halo = 0, tables = 0;
    for (uint64_t g = 0; g < G; ++g) {
        if (sj[g] == cdc::SJ_TABLE) ++tables;
        if (sj[g] == (int32_t)(g + 1) || sj[g] == cdc::SJ_LAST || sj[g] == cdc::SJ_TABLE) ++met;
        else if (sj[g] == cdc::SJ_UNSYNCED) ++unsynced;
        else ++other;
        halo += hc[g];
    }
    stats[0] = G;
    stats[1] = P.S;
    stats[2] = P.Hmax;
    stats[3] = ctrl[1] == 0 ? 0 : (tables == G && G > 0 ? 2 : 1);
    if (getenv("CDC_TDEBUG")) {  // why the transfer tables gave up (diagnostics)
        uint32_t why[5] = {0, 0, 0, 0, 0}, lim = 0;
        CDC_CUDA(cudaMemcpy(why, W.ctrl + 11, 20, cudaMemcpyDeviceToHost));
        CDC_CUDA(cudaMemcpy(&lim, W.ctrl + 10, 4, cudaMemcpyDeviceToHost));
        fprintf(stderr, "cdc: transfer tables: hand-over limits word %08x\n", lim + 1u);
        fprintf(stderr,
                "cdc: transfer tables: reason %d at segment %u; unresolved chains: %d over their byte-step budget, "
                "%d extra entries past the next segment, %d hand-overs that did not fit\n",
                (int)why[1], why[2], (int)(why[3] + 1), (int)(why[0] + 1), (int)(why[4] + 1));
    }
    stats[4] = met;
    stats[5] = unsynced;
    stats[6] = other;
    stats[7] = halo;
    return CDC_OK;
}

int cdc_profile_query(int *done) {
    // completion state of the events of the last profiled call (1 = reached)
    if (!done) return fail(CDC_ERR_INVALID, "null");
    if (g_prof_calls.empty()) return fail(CDC_ERR_INVALID, "no profiled call");
    ProfCall &pc = g_prof_calls.back();
    for (int k = 0; k <= PROF_KERNELS; ++k) done[k] = pc.ev[k] ? (cudaEventQuery(pc.ev[k]) == cudaSuccess) : -1;
    return CDC_OK;
}

int cdc_profile_enable(int on) {
    g_prof_on = on != 0;
    return CDC_OK;
}

int cdc_profile_collect(double *ms_sum, uint64_t *launches, uint64_t *calls) {
    if (!ms_sum || !launches || !calls) return fail(CDC_ERR_INVALID, "null pointer");
    for (int k = 0; k < PROF_KERNELS; ++k) {
        ms_sum[k] = 0.0;
        launches[k] = 0;
    }
    *calls = g_prof_calls.size();
    for (ProfCall &pc : g_prof_calls) {
        CDC_CUDA(cudaEventSynchronize(pc.ev[PROF_KERNELS]));
        for (int k = 0; k < PROF_KERNELS; ++k) {
            if (!pc.used[k]) continue;
            float ms = 0.f;
            CDC_CUDA(cudaEventElapsedTime(&ms, pc.ev[k], pc.ev[k + 1]));
            ms_sum[k] += ms;
            launches[k] += 1;
        }
        for (int k = 0; k <= PROF_KERNELS; ++k) g_prof_pool.push_back(pc.ev[k]);
    }
    g_prof_calls.clear();
    return CDC_OK;
}

int cdc_window_for_avg(int32_t algo, uint64_t avg_size, uint32_t *window) {
    if (!window) return fail(CDC_ERR_INVALID, "null window");
    if (algo < CDC_RAM || algo > CDC_MAXP) return fail(CDC_ERR_INVALID, "unknown algorithm");
    if (avg_size < 2 || avg_size > (1ull << 31)) return fail(CDC_ERR_INVALID, "avg_size out of range");
    if (algo == CDC_MAXP) {
        // reading M5: on i.i.d. uniform bytes a byte is a strict maximum of its 2h
        // neighbours with probability P(h) = sum_v (1/256) (v/256)^(2h); local maxima
        // (the chunk ends) are then 1/P(h) bytes apart on average: the smallest h
        // with 1/P(h) >= avg (at most MX_HMAX)
        uint32_t h = 1;
        for (; h < cdc::MX_HMAX; ++h) {
            double pr = 0.0;
            for (int v = 1; v < 256; ++v) pr += std::pow(v / 256.0, 2.0 * h);
            if (256.0 / pr >= (double)avg_size) break;
        }
        *window = h;
        return CDC_OK;
    }
    *window = (uint32_t)(avg_size >= 512 ? avg_size - 256 : avg_size / 2);
    return CDC_OK;
}

int cdc_params_default(cdc_params *p, int32_t algo, uint64_t avg_size) {
    if (!p) return fail(CDC_ERR_INVALID, "null params");
    uint32_t w;
    int rc = cdc_window_for_avg(algo, avg_size, &w);
    if (rc) return rc;
    p->algo = algo;
    p->window = w;
    p->max_size = 4 * avg_size;
    p->seg_bytes = 0;
    p->halo_bytes = 0;
    return CDC_OK;
}

uint64_t cdc_max_boundaries(const cdc_params *p, uint64_t len) {
    if (!p || p->window < 1) return 0;
    return len / ((uint64_t)p->window + 1) + 1;
}

int cdc_workspace_size(const cdc_params *p, uint64_t nfiles, uint64_t total_len, uint64_t max_len, size_t *bytes) {
    int rc = check_params(p);
    if (rc) return rc;
    if (!bytes) return fail(CDC_ERR_INVALID, "null bytes");
    if (p->algo == CDC_MAXP) {
        MaxpPlan M;
        maxp_plan(p, nfiles ? nfiles : 1, total_len, M);
        *bytes = M.bytes;
        return CDC_OK;
    }
    Plan P;
    make_plan(p, nfiles ? nfiles : 1, total_len, max_len, P);
    *bytes = P.bytes;
    return CDC_OK;
}

int cdc_chunk(const cdc_params *p, const uint8_t *d_data, uint64_t len, uint64_t *d_bounds, uint64_t bounds_cap,
              uint64_t *d_count, void *d_workspace, size_t workspace_bytes, void *stream) {
    return run_chunk(p, d_data, nullptr, 1, len, len, d_bounds, bounds_cap, nullptr, d_count, d_workspace,
                     workspace_bytes, stream, false);
}

int cdc_chunk_batch(const cdc_params *p, const uint8_t *d_data, const uint64_t *d_file_offsets, uint64_t nfiles,
                    uint64_t total_len, uint64_t max_len, uint64_t *d_bounds, uint64_t bounds_cap,
                    uint64_t *d_bound_offsets, uint64_t *d_count, void *d_workspace, size_t workspace_bytes,
                    void *stream) {
    if (!d_file_offsets || !d_bound_offsets) return fail(CDC_ERR_INVALID, "null offsets");
    if (nfiles == 0) return fail(CDC_ERR_INVALID, "nfiles must be >= 1");
    return run_chunk(p, d_data, d_file_offsets, nfiles, total_len, max_len, d_bounds, bounds_cap, d_bound_offsets,
                     d_count, d_workspace, workspace_bytes, stream, true);
}

int cdc_chunk_host(const cdc_params *p, const uint8_t *h_data, uint64_t len, uint64_t *h_bounds,
                   uint64_t bounds_cap, uint64_t *h_count) {
    int rc = check_params(p);
    if (rc) return rc;
    if ((!h_data && len) || !h_count || (!h_bounds && bounds_cap)) return fail(CDC_ERR_INVALID, "null pointer");
    HostCache *Cp = nullptr;
    if ((rc = host_cache(Cp))) return rc;
    HostCache &C = *Cp;
    size_t wsb = 0;
    if ((rc = cdc_workspace_size(p, 1, len, len, &wsb))) return rc;
    const uint64_t maxb = cdc_max_boundaries(p, len);
    if ((rc = ensure((void **)&C.data, C.data_cap, len + 32))) return rc;
    if ((rc = ensure((void **)&C.bounds, C.bounds_cap, maxb * 8))) return rc;
    if ((rc = ensure(&C.ws, C.ws_cap, wsb))) return rc;
    CDC_CUDA(cudaMemcpyAsync(C.data, h_data, len, cudaMemcpyHostToDevice, C.st));
    if ((rc = cdc_chunk(p, C.data, len, C.bounds, maxb, C.count, C.ws, C.ws_cap, C.st))) return rc;
    uint64_t n = 0;
    CDC_CUDA(cudaMemcpyAsync(&n, C.count, 8, cudaMemcpyDeviceToHost, C.st));
    CDC_CUDA(cudaStreamSynchronize(C.st));
    *h_count = n;
    const uint64_t m = n < bounds_cap ? n : bounds_cap;
    if (m) {
        CDC_CUDA(cudaMemcpyAsync(h_bounds, C.bounds, m * 8, cudaMemcpyDeviceToHost, C.st));
        CDC_CUDA(cudaStreamSynchronize(C.st));
    }
    if (n > bounds_cap) return fail(CDC_ERR_CAPACITY, "bounds_cap too small");
    return CDC_OK;
}

int cdc_plan_segments(const cdc_params *p, uint64_t len, uint64_t *starts, uint64_t starts_cap, uint64_t *n_out) {
    int rc = check_params(p);
    if (rc) return rc;
    if (p->algo == CDC_MAXP) return fail(CDC_ERR_INVALID, "not defined for MAXP (no speculative segments)");
    if (!n_out || (!starts && starts_cap)) return fail(CDC_ERR_INVALID, "null pointer");
    Plan P;
    make_plan(p, 1, len, len, P);
    const uint64_t n = cdc::nseg_of(len, P.S);
    *n_out = n;
    for (uint64_t k = 0; k < n && k < starts_cap; ++k) starts[k] = (uint64_t)cdc::seg_start(k, n, len);
    return CDC_OK;
}

int cdc_chunk_batch_host(const cdc_params *p, const uint8_t *h_data, const uint64_t *h_file_offsets,
                         uint64_t nfiles, uint64_t *h_bounds, uint64_t bounds_cap, uint64_t *h_bound_offsets,
                         uint64_t *h_count) {
    int rc = check_params(p);
    if (rc) return rc;
    if (!h_file_offsets || !h_bound_offsets || !h_count || (!h_bounds && bounds_cap))
        return fail(CDC_ERR_INVALID, "null pointer");
    if (nfiles == 0) return fail(CDC_ERR_INVALID, "nfiles must be >= 1");
    const uint64_t total = h_file_offsets[nfiles] - h_file_offsets[0];
    if (total && !h_data) return fail(CDC_ERR_INVALID, "null data");
    for (uint64_t f = 0; f < nfiles; ++f)
        if (h_file_offsets[f + 1] < h_file_offsets[f]) return fail(CDC_ERR_INVALID, "file offsets decrease");
    HostCache *Cp = nullptr;
    if ((rc = host_cache(Cp))) return rc;
    HostCache &C = *Cp;
    // groups of whole files of about total / ngroups bytes each: group k's copy
    // overlaps group k-1's chunking
    const uint64_t ngroups_want = std::min<uint64_t>(
        std::max<uint64_t>(total / CDC_HOST_GROUP_BYTES, 1), CDC_HOST_GROUPS_MAX);
    std::vector<uint64_t> gf{0};  // first file of each group
    for (uint64_t k = 1; k < ngroups_want; ++k) {
        const uint64_t target = h_file_offsets[0] + total / ngroups_want * k;
        uint64_t lo = gf.back(), hi = nfiles;  // first file starting at or after target
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if (h_file_offsets[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        if (lo > gf.back() && lo < nfiles) gf.push_back(lo);
    }
    gf.push_back(nfiles);
    const size_t ng = gf.size() - 1;
    // per-group plan: workspace, bound capacity (every chunk but a file's last holds > w bytes)
    const uint64_t w1 = (uint64_t)p->window + 1;
    std::vector<uint64_t> gb(ng + 1, 0), gmax(ng, 0), gcap(ng + 1, 0);
    size_t ws_max = 0;
    for (size_t k = 0; k < ng; ++k) {
        uint64_t mx = 0, cap = 0;
        for (uint64_t f = gf[k]; f < gf[k + 1]; ++f) {
            const uint64_t L = h_file_offsets[f + 1] - h_file_offsets[f];
            mx = std::max(mx, L);
            cap += L / w1 + 1;
        }
        gb[k + 1] = h_file_offsets[gf[k + 1]] - h_file_offsets[0];
        gmax[k] = mx;
        gcap[k + 1] = gcap[k] + cap;
        size_t wsb = 0;
        if ((rc = cdc_workspace_size(p, gf[k + 1] - gf[k], gb[k + 1] - gb[k], mx, &wsb))) return rc;
        ws_max = std::max(ws_max, round_up(wsb, 256));
    }
    if ((rc = ensure((void **)&C.data, C.data_cap, total + 32))) return rc;
    if ((rc = ensure((void **)&C.bounds, C.bounds_cap, std::max<uint64_t>(gcap[ng], 1) * 8))) return rc;
    if ((rc = ensure(&C.ws, C.ws_cap, ws_max))) return rc;
    if ((rc = ensure((void **)&C.offs, C.offs_cap, (nfiles + ng) * 8))) return rc;
    if ((rc = ensure((void **)&C.bo, C.bo_cap, (nfiles + ng) * 8))) return rc;
    // rebased offsets of every group (host staging, then one copy)
    std::vector<uint64_t> ro(nfiles + ng);
    for (size_t k = 0; k < ng; ++k)
        for (uint64_t f = gf[k]; f <= gf[k + 1]; ++f) ro[f + k] = h_file_offsets[f] - h_file_offsets[gf[k]];
    CDC_CUDA(cudaMemcpyAsync(C.offs, ro.data(), ro.size() * 8, cudaMemcpyHostToDevice, C.cp));
    for (size_t k = 0; k < ng; ++k) {
        const uint64_t nb = gb[k + 1] - gb[k];
        if (nb)
            CDC_CUDA(cudaMemcpyAsync(C.data + gb[k], h_data + h_file_offsets[gf[k]], nb, cudaMemcpyHostToDevice,
                                     C.cp));
        CDC_CUDA(cudaEventRecord(C.ev[k], C.cp));
    }
    int launches = 0;
    for (size_t k = 0; k < ng; ++k) {
        CDC_CUDA(cudaStreamWaitEvent(C.st, C.ev[k], 0));
        const uint64_t nf = gf[k + 1] - gf[k];
        // one workspace: the groups' pipelines are ordered on the compute stream
        if ((rc = cdc_chunk_batch(p, C.data + gb[k], C.offs + gf[k] + k, nf, gb[k + 1] - gb[k], gmax[k],
                                  C.bounds + gcap[k], gcap[k + 1] - gcap[k], C.bo + gf[k] + k, C.count + 1 + k, C.ws,
                                  C.ws_cap, C.st)))
            return rc;
        launches += g_launches;
    }
    // per-group bound offsets back to the host, then the boundaries of each group
    std::vector<uint64_t> hbo(nfiles + ng);
    CDC_CUDA(cudaMemcpyAsync(hbo.data(), C.bo, hbo.size() * 8, cudaMemcpyDeviceToHost, C.st));
    CDC_CUDA(cudaStreamSynchronize(C.st));
    uint64_t n = 0;
    for (size_t k = 0; k < ng; ++k) {
        const uint64_t nf = gf[k + 1] - gf[k];
        const uint64_t *b = hbo.data() + gf[k] + k;
        const uint64_t m = b[nf];
        if (m > gcap[k + 1] - gcap[k]) return fail(CDC_ERR_CUDA, "internal: group bound capacity exceeded");
        for (uint64_t i = 0; i < nf; ++i) h_bound_offsets[gf[k] + i] = n + b[i];
        const uint64_t room = n < bounds_cap ? bounds_cap - n : 0;
        const uint64_t mm = m < room ? m : room;
        if (mm) CDC_CUDA(cudaMemcpyAsync(h_bounds + n, C.bounds + gcap[k], mm * 8, cudaMemcpyDeviceToHost, C.st));
        n += m;
    }
    h_bound_offsets[nfiles] = n;
    *h_count = n;
    CDC_CUDA(cudaStreamSynchronize(C.st));
    g_launches = launches;
    if (n > bounds_cap) return fail(CDC_ERR_CAPACITY, "bounds_cap too small");
    return CDC_OK;
}

int cdc_chain(const cdc_params *p, const uint8_t *d_data, uint64_t len, uint64_t start, uint64_t stop,
              uint64_t *d_starts, uint64_t starts_cap, uint64_t *d_count, void *stream) {
    int rc = check_params(p);
    if (rc) return rc;
    if (p->algo == CDC_MAXP) return fail(CDC_ERR_INVALID, "not defined for MAXP (no speculative segments)");
    if (!d_count || (!d_starts && starts_cap) || (!d_data && len)) return fail(CDC_ERR_INVALID, "null pointer");
    if (start > len) return fail(CDC_ERR_INVALID, "start beyond len");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static bool attr[MAX_DEVICES] = {false};
    const int dev = current_device();
    if (!attr[dev]) {
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_chain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, cdc::RING_SMEM + 128));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, cdc::RING_SMEM + 128));
        CDC_CUDA(cudaFuncSetAttribute(cdc::k_chain<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cdc::RING_SMEM + 128));
        attr[dev] = true;
    }
    switch (p->algo) {
    case CDC_RAM:
        cdc::k_chain<0><<<1, 32, cdc::RING_SMEM + 128, st>>>(d_data, len, start, stop, p->window, p->max_size, d_starts,
                                                       starts_cap, d_count, sparse_on(p->window, p->max_size));
        break;
    case CDC_AE_MAX:
        cdc::k_chain<1><<<1, 32, cdc::RING_SMEM + 128, st>>>(d_data, len, start, stop, p->window, p->max_size, d_starts,
                                                       starts_cap, d_count, sparse_on(p->window, p->max_size));
        break;
    default:
        cdc::k_chain<2><<<1, 32, cdc::RING_SMEM + 128, st>>>(d_data, len, start, stop, p->window, p->max_size, d_starts,
                                                       starts_cap, d_count, sparse_on(p->window, p->max_size));
    }
    g_launches = 1;
    CDC_CUDA(cudaGetLastError());
    return CDC_OK;
}

int cdc_first_common(const int64_t *d_a, uint64_t na, const int64_t *d_b, uint64_t nb, int64_t *d_out,
                     void *stream) {
    if (!d_out || (na && !d_a) || (nb && !d_b)) return fail(CDC_ERR_INVALID, "null pointer");
    if (na >= (1ull << 32) || nb >= (1ull << 32)) return fail(CDC_ERR_INVALID, "lists longer than 2^32 entries");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cdc::k_first_common<<<1, 1024, 0, st>>>(d_a, na, d_b, nb, d_out);
    g_launches = 1;
    CDC_CUDA(cudaGetLastError());
    return CDC_OK;
}

int cdc_extreme_byte_search(const uint8_t *d_data, const uint64_t *d_off, const uint64_t *d_len, uint64_t n,
                            int32_t mode, uint8_t *d_value, uint64_t *d_pos, void *stream) {
    if (n == 0) return CDC_OK;
    if (!d_data || !d_off || !d_len || !d_value || !d_pos) return fail(CDC_ERR_INVALID, "null pointer");
    if (mode != CDC_EXT_MAX && mode != CDC_EXT_MIN) return fail(CDC_ERR_INVALID, "bad mode");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned blocks = (unsigned)((n * 32 + 255) / 256);
    if (mode == CDC_EXT_MAX) cdc::k_ebs<true><<<blocks, 256, 0, st>>>(d_data, d_off, d_len, n, d_value, d_pos);
    else cdc::k_ebs<false><<<blocks, 256, 0, st>>>(d_data, d_off, d_len, n, d_value, d_pos);
    g_launches = 1;
    CDC_CUDA(cudaGetLastError());
    return CDC_OK;
}

int cdc_range_scan(const uint8_t *d_data, const uint64_t *d_off, const uint64_t *d_len, const uint8_t *d_target,
                   uint64_t n, int32_t cmp, uint64_t *d_pos, void *stream) {
    if (n == 0) return CDC_OK;
    if (!d_data || !d_off || !d_len || !d_target || !d_pos) return fail(CDC_ERR_INVALID, "null pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned blocks = (unsigned)((n * 32 + 255) / 256);
    switch (cmp) {
    case CDC_GT: cdc::k_range_scan<cdc::CMP_GT><<<blocks, 256, 0, st>>>(d_data, d_off, d_len, d_target, n, d_pos); break;
    case CDC_GEQ: cdc::k_range_scan<cdc::CMP_GEQ><<<blocks, 256, 0, st>>>(d_data, d_off, d_len, d_target, n, d_pos); break;
    case CDC_LT: cdc::k_range_scan<cdc::CMP_LT><<<blocks, 256, 0, st>>>(d_data, d_off, d_len, d_target, n, d_pos); break;
    case CDC_LEQ: cdc::k_range_scan<cdc::CMP_LEQ><<<blocks, 256, 0, st>>>(d_data, d_off, d_len, d_target, n, d_pos); break;
    case CDC_EQ: cdc::k_range_scan<cdc::CMP_EQ><<<blocks, 256, 0, st>>>(d_data, d_off, d_len, d_target, n, d_pos); break;
    default: return fail(CDC_ERR_INVALID, "bad comparator");
    }
    g_launches = 1;
    CDC_CUDA(cudaGetLastError());
    return CDC_OK;
}

}  // extern "C"
