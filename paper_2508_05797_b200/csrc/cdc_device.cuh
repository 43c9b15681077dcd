// cdc_device.cuh -- device building blocks of the sm_100a chunker.
//
//  * PTX wrappers: mbarrier, 1-D TMA bulk copy (cp.async.bulk -> UBLKCP),
//    L2 evict-first policy, acquire/release flags.
//  * Byte SIMD on 16-byte lane vectors: Extreme Byte Search (§4.1)
//    as a max/min tree over the lane's 16 bytes with the native DPX
//    VIMNMX3.U16x2 instruction, rooted in a warp CREDUX reduction; Range Scan
//    (§4.2) as a per-lane "any byte satisfies" test, a warp ballot and __ffs,
//    then one in-lane byte locate -- the GPU form of the paper's VCMP + VMASK
//    "packed scanning".
//  * run_chain: one warp walks the chunk chain of one stream from a given
//    start, streaming the bytes through a private shared-memory ring of NST
//    STAGE-byte stages filled by TMA.  RAM (§2.1.2 l.198; §4.3 l.355) and
//    AE-Max / AE-Min (§2.1.2 l.169-171; §4.3 l.357-359) are block-granular
//    state machines: each 512-byte warp block (32 lanes x 16 B) is loaded from
//    shared memory once, its per-lane extreme is computed once, and every
//    event inside the block (window end, boundary, new AE target) costs O(1)
//    warp operations.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cdc {

constexpr int BLK = 512;               // bytes per warp block: 32 lanes x 16 B
#ifndef CDC_YIELD_SAT
#define CDC_YIELD_SAT 2
#endif
constexpr int YIELD_SAT = CDC_YIELD_SAT;  // saturated chunks after which the ring walker yields to the sparse walk
#ifndef CDC_STAGE
#define CDC_STAGE 6144
#endif
#ifndef CDC_NST
#define CDC_NST 2
#endif
constexpr int STAGE = CDC_STAGE;       // bytes per TMA stage (12 warp blocks)
constexpr int NST = CDC_NST;           // ring depth per warp (12 KiB)
constexpr int RING_BYTES = STAGE * NST;
constexpr int RING_SMEM = (RING_BYTES + NST * 8 + 127) / 128 * 128;  // keeps every ring 128-byte aligned
// R.bar[FETCH_SLOT]: bytes this warp's bulk copies fetched (ring stages and
// sparse-walk regions), flushed into the workspace by k_speculate (cdc_fetched)
constexpr int FETCH_SLOT = 5;
static_assert(RING_BYTES + 8 * (FETCH_SLOT + 1) <= RING_SMEM, "fetch counter after the ring's mbarriers");
// A ring of NST stages of STG bytes (the default is STAGE; the batch kernel
// uses a smaller one so that more walkers fit an SM): its bytes and its
// shared-memory stride (bytes + mbarriers + fetch counter, 128-byte aligned).
template <int STG>
struct Ring {
    static constexpr int BYTES = STG * NST;
    static constexpr int SMEM = (BYTES + 8 * (FETCH_SLOT + 1) + 127) / 128 * 128;
};
static_assert(Ring<STAGE>::SMEM == RING_SMEM, "default ring stride");

enum { ALGO_RAM = 0, ALGO_AE_MAX = 1, ALGO_AE_MIN = 2 };
enum { CMP_GT = 0, CMP_GEQ = 1, CMP_LT = 2, CMP_LEQ = 3, CMP_EQ = 4 };

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_inval(uint64_t *bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Watchdog: a stage that has not landed within ~10 s (clock64) means a lost
// bulk copy; trap instead of hanging the GPU.
__device__ unsigned long long g_wait_ns = 0;  // diagnostic: total ns spent waiting for stages (CDC_WAIT_PROBE)
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#ifdef CDC_WAIT_PROBE
    unsigned long long t0g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0g));
    while (!mbar_try_wait(bar, parity)) {
    }
    unsigned long long t1g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1g));
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_wait_ns, t1g - t0g);
    return;
#endif
    if (mbar_try_wait(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, parity)) {
        if (clock64() - t0 > 20000000000ll) __trap();
    }
}
// the same on a 32-bit shared-window address (the sparse walk keeps its ring's)
__device__ __forceinline__ bool mbar_try_wait_s(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_s(uint32_t a, uint32_t parity) {
    if (mbar_try_wait_s(a, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait_s(a, parity)) {
        if (clock64() - t0 > 20000000000ll) __trap();
    }
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Diagnostic per-warp cycle accounting (CDC_EVTIME builds only): ET_BEGIN(v)
// stamps clock64, ET_ADD(i, v) adds the cycles since the stamp to bucket i.
__device__ unsigned long long g_evt[16];
#ifdef CDC_EVTIME
#define ET_DECL long long et_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long et_t0 = clock64(), et_t1 = 0, et_h0 = 0, et_hs = 0;
// halo phase (emitter past its segment end): bucket 7 = its stage transitions,
// g_evt[9] = its stages, g_evt[10] = its cycles
#define ET_HALO_STAGE(h, v)                          \
    if (h) {                                         \
        if (et_h0 == 0) et_h0 = v;                   \
        et_acc[7] += clock64() - v;                  \
        ++et_hs;                                     \
    }
#define ET_VAR(v) long long v;
#define ET_BEGIN(v) v = clock64()
#define ET_ADD(i, v) et_acc[i] += clock64() - v
#define ET_FLUSH                                                        \
    if ((threadIdx.x & 31) == 0) {                                      \
        for (int q = 0; q < 8; ++q) atomicAdd(&g_evt[q], (unsigned long long)et_acc[q]); \
        atomicAdd(&g_evt[8], (unsigned long long)(clock64() - et_t0));  \
        atomicAdd(&g_evt[9], (unsigned long long)et_hs);                \
        if (et_h0) atomicAdd(&g_evt[10], (unsigned long long)(clock64() - et_h0)); \
    }
#else
#define ET_HALO_STAGE(h, v)
#define ET_DECL
#define ET_VAR(v)
#define ET_BEGIN(v)
#define ET_ADD(i, v)
#define ET_FLUSH
#endif

// Diagnostic event counters (CDC_COUNTERS builds only): CNT(i) adds 1 per warp.
__device__ unsigned long long g_cnt[16];
#ifdef CDC_COUNTERS
#define CNT(i)                                              \
    do {                                                    \
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_cnt[i], 1ull); \
    } while (0)
#else
#define CNT(i) \
    do {       \
    } while (0)
#endif

// ---------------------------------------------------------------- byte SIMD
// Extreme of bytes with the DPX 3-input u16x2 min/max: the high byte of the
// u16 extreme of a set of 16-bit halves is the extreme of their high bytes,
// whatever the low bytes are.  A word's halves carry bytes 1 and 3 in their
// high bytes; the word shifted left by 8 carries bytes 0 and 2 there.
template <bool MAX>
__device__ __forceinline__ uint32_t ext3(uint32_t a, uint32_t b, uint32_t c) {
    if constexpr (MAX)
        return __vimax3_u16x2(a, b, c);
    else
        return __vimin3_u16x2(a, b, c);
}
template <bool MAX>
__device__ __forceinline__ uint32_t neutral() {
    return MAX ? 0u : 255u;
}
template <bool MAX>
__device__ __forceinline__ uint32_t ext2(uint32_t a, uint32_t b) {
    return MAX ? max(a, b) : min(a, b);
}
template <bool MAX>
__device__ __forceinline__ bool beats(uint32_t a, uint32_t b) {  // a strictly more extreme than b
    return MAX ? a > b : a < b;
}
// extreme byte of a 16-byte vector (Extreme Byte Search, §4.1, one tree leaf)
template <bool MAX>
__device__ __forceinline__ uint32_t vext16(const uint4 &v) {
    const uint32_t a = ext3<MAX>(v.x, v.y, v.z);
    const uint32_t b = ext3<MAX>(v.w, v.x << 8, v.y << 8);
    const uint32_t c = ext3<MAX>(v.z << 8, v.w << 8, a);
    const uint32_t m = ext3<MAX>(b, c, c);
    return ext2<MAX>(m >> 24, (m >> 8) & 0xFFu);
}
// byte mask (0xFF for kept bytes) of bytes [lo, hi) of the word holding bytes [4j, 4j+4)
__device__ __forceinline__ uint32_t word_keep(int lo, int hi, int j) {
    int a = lo - 4 * j, z = hi - 4 * j;
    a = a < 0 ? 0 : (a > 4 ? 4 : a);
    z = z < 0 ? 0 : (z > 4 ? 4 : z);
    const uint32_t up = z >= 4 ? 0xFFFFFFFFu : ((1u << (8 * z)) - 1u);
    const uint32_t dn = a >= 4 ? 0xFFFFFFFFu : ((1u << (8 * a)) - 1u);
    return up & ~dn;
}
// extreme byte of bytes [lo, hi) of a 16-byte vector (0 <= lo < hi <= 16)
template <bool MAX>
__device__ __forceinline__ uint32_t vext16_range(const uint4 &v, int lo, int hi) {
    uint4 r;
    const uint32_t k0 = word_keep(lo, hi, 0), k1 = word_keep(lo, hi, 1), k2 = word_keep(lo, hi, 2),
                   k3 = word_keep(lo, hi, 3);
    if (MAX) {
        r.x = v.x & k0; r.y = v.y & k1; r.z = v.z & k2; r.w = v.w & k3;
    } else {
        r.x = v.x | ~k0; r.y = v.y | ~k1; r.z = v.z | ~k2; r.w = v.w | ~k3;
    }
    return vext16<MAX>(r);
}
template <bool MAX>
__device__ __forceinline__ uint32_t warp_ext(uint32_t v) {
    if constexpr (MAX)
        return __reduce_max_sync(0xFFFFFFFFu, v);
    else
        return __reduce_min_sync(0xFFFFFFFFu, v);
}
// byte j (0..15) of a 16-byte vector
__device__ __forceinline__ uint32_t vbyte(const uint4 &v, int j) {
    const int q = j >> 2;
    const uint32_t wd = q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
    return (wd >> (8 * (j & 3))) & 0xFFu;
}

template <int CMP>
__device__ __forceinline__ bool cmp_holds(uint32_t b, uint32_t t) {
    if constexpr (CMP == CMP_GT) return b > t;
    else if constexpr (CMP == CMP_GEQ) return b >= t;
    else if constexpr (CMP == CMP_LT) return b < t;
    else if constexpr (CMP == CMP_LEQ) return b <= t;
    else return b == t;
}

// Lane-vector view of one 512-byte block of the ring: lane l holds bytes
// [16 l, 16 l + 16) of the block in v, their extreme in full (computed once).
struct Blk {
    uint4 v;
    int64_t B;  // stream position of the block's byte 0
};
// lane's part [a, b) (0..16) of the block range [rlo, rhi) (block-relative)
__device__ __forceinline__ void lane_part(int rlo, int rhi, int &a, int &b) {
    const int base = lane_id() * 16;
    a = rlo - base;
    b = rhi - base;
    a = a < 0 ? 0 : (a > 16 ? 16 : a);
    b = b < 0 ? 0 : (b > 16 ? 16 : b);
}
// per-lane extreme of the block range [rlo, rhi); `full` is the lane's
// whole-vector extreme; `has` tells whether the lane holds any byte of the range
// (lanes without one return the neutral value and must not join a ballot).
template <bool MAX>
__device__ __forceinline__ uint32_t lane_ext(const Blk &k, uint32_t full, int rlo, int rhi, bool &has) {
    int a, b;
    lane_part(rlo, rhi, a, b);
    has = a < b;
    if (a == 0 && b == 16) return full;
    if (a >= b) return neutral<MAX>();
    return vext16_range<MAX>(k.v, a, b);
}
// Range Scan locate (§4.2): first block-relative index in [rlo, rhi) whose byte
// satisfies (byte CMP target), given the ballot `bal` of lanes that hold one.
template <int CMP>
__device__ __forceinline__ int locate(const Blk &k, uint32_t bal, int rlo, int rhi, uint32_t target) {
    const int L = __ffs(bal) - 1;
    uint4 u;
    u.x = __shfl_sync(0xFFFFFFFFu, k.v.x, L);
    u.y = __shfl_sync(0xFFFFFFFFu, k.v.y, L);
    u.z = __shfl_sync(0xFFFFFFFFu, k.v.z, L);
    u.w = __shfl_sync(0xFFFFFFFFu, k.v.w, L);
    const int j = lane_id() & 15;
    const int pos = L * 16 + j;
    const bool hit = lane_id() < 16 && pos >= rlo && pos < rhi && cmp_holds<CMP>(vbyte(u, j), target);
    const uint32_t b2 = __ballot_sync(0xFFFFFFFFu, hit);
    return L * 16 + __ffs(b2) - 1;
}

// ---------------------------------------------------------------- warp ring
struct WarpRing {
    uint8_t *buf;   // NST * STAGE bytes, 128-byte aligned
    uint64_t *bar;  // NST mbarriers
};

// ---------------------------------------------------------------- chain engine
//
// L2 policies of the ring's bulk copies: bytes below keep_until (a segment's
// head, which the previous segment's halo walk reads again) are loaded with
// `keep`, the rest with `stream` (evict-first: read once).
struct L2Pol {
    uint64_t stream, keep;
    int64_t keep_until;
};
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ L2Pol stream_policy() { return L2Pol{l2_evict_first_policy(), 0, INT64_MIN}; }

// ---------------------------------------------------------------- stage scans
// Per-lane extreme of bytes [lo, hi) (stage offsets, lo < hi) of the 512-byte
// block at stage offset Bk; `has` = the lane holds a byte of the range.
template <bool MAX>
__device__ __forceinline__ uint32_t block_lane_ext(const uint8_t *sp, int Bk, int lo, int hi, bool &has,
                                                   uint4 &v) {
    // branch-free: a 16-bit keep mask of the lane's bytes in [lo, hi), expanded
    // to byte masks; bytes outside become the neutral value
    v = *reinterpret_cast<const uint4 *>(sp + Bk + lane_id() * 16);
    int a, b;
    lane_part(lo - Bk, hi - Bk, a, b);
    has = a < b;
    const uint32_t m16 = has ? (((1u << b) - 1u) & ~((1u << a) - 1u)) : 0u;
    auto expand = [](uint32_t nib) { return ((nib * 0x00204081u) & 0x01010101u) * 0xFFu; };
    const uint32_t k0 = expand(m16 & 0xFu), k1 = expand((m16 >> 4) & 0xFu), k2 = expand((m16 >> 8) & 0xFu),
                   k3 = expand(m16 >> 12);
    uint4 r;
    if (MAX) {
        r.x = v.x & k0; r.y = v.y & k1; r.z = v.z & k2; r.w = v.w & k3;
    } else {
        r.x = v.x | ~k0; r.y = v.y | ~k1; r.z = v.z | ~k2; r.w = v.w | ~k3;
    }
    return vext16<MAX>(r);
}


// RAM window (Extreme Byte Search, §4.1) with early saturation: folds the
// per-lane max of the stage bytes [lo, hi) into acc, and stops as soon as some
// byte equals 255 -- no byte can exceed it, so the window's maximum is known
// and the rest of the window need not be read.  Returns true when saturated.
__device__ __forceinline__ bool stage_window_max(const uint8_t *sp, int lo, int hi, uint32_t &acc) {
    const int lane16 = lane_id() * 16;
    int Bk = lo & ~(BLK - 1);
    uint4 v;
    bool has;
    if (Bk < lo || Bk + BLK > hi) {  // partial head block
        if (Bk >= hi) return false;
        const uint32_t lm = block_lane_ext<true>(sp, Bk, lo, hi < Bk + BLK ? hi : Bk + BLK, has, v);
        acc = max(acc, lm);
        if (__any_sync(0xFFFFFFFFu, lm == 255u)) return true;
        Bk += BLK;
    }
    for (; Bk + 2 * BLK <= hi; Bk += 2 * BLK) {
        const uint4 a = *reinterpret_cast<const uint4 *>(sp + Bk + lane16);
        const uint4 b = *reinterpret_cast<const uint4 *>(sp + Bk + BLK + lane16);
        const uint32_t m = max(vext16<true>(a), vext16<true>(b));
        acc = max(acc, m);
        if (__any_sync(0xFFFFFFFFu, m == 255u)) return true;
    }
    for (; Bk + BLK <= hi; Bk += BLK) {
        v = *reinterpret_cast<const uint4 *>(sp + Bk + lane16);
        const uint32_t m = vext16<true>(v);
        acc = max(acc, m);
        if (__any_sync(0xFFFFFFFFu, m == 255u)) return true;
    }
    if (Bk < hi) {  // partial tail block
        const uint32_t lm = block_lane_ext<true>(sp, Bk, Bk, hi, has, v);
        acc = max(acc, lm);
        if (__any_sync(0xFFFFFFFFu, lm == 255u)) return true;
    }
    return false;
}

// Range Scan (§4.2), block level: first 512-byte block of the stage bytes
// [lo, hi) holding a byte b with (b CMP target).  Returns its stage offset Bk
// (or -1), the ballot of the lanes holding one, and each lane's extreme `lm`
// (and `has`) over that block's part of [lo, hi).  Whole blocks are tested two
// at a time (two independent shared-memory loads and max trees in flight).
template <int CMP>
__device__ __forceinline__ int stage_find_block(const uint8_t *sp, int lo, int hi, uint32_t target, uint32_t &bal,
                                                uint32_t &lm, bool &has) {
    constexpr bool MAX = (CMP == CMP_GT || CMP == CMP_GEQ);
    const int lane16 = lane_id() * 16;
    int Bk = lo & ~(BLK - 1);
    uint4 v;
    CNT(7);
    if (Bk < lo || Bk + BLK > hi) {  // partial head block
        if (Bk >= hi) return -1;
        CNT(9);
        lm = block_lane_ext<MAX>(sp, Bk, lo, hi < Bk + BLK ? hi : Bk + BLK, has, v);
        bal = __ballot_sync(0xFFFFFFFFu, has && cmp_holds<CMP>(lm, target));
        if (bal) return Bk;
        Bk += BLK;
    }
    has = true;
    for (; Bk + 4 * BLK <= hi; Bk += 4 * BLK) {  // four blocks in flight
        const uint4 a = *reinterpret_cast<const uint4 *>(sp + Bk + lane16);
        const uint4 b = *reinterpret_cast<const uint4 *>(sp + Bk + BLK + lane16);
        const uint4 c = *reinterpret_cast<const uint4 *>(sp + Bk + 2 * BLK + lane16);
        const uint4 d = *reinterpret_cast<const uint4 *>(sp + Bk + 3 * BLK + lane16);
        const uint32_t ma = vext16<MAX>(a), mb = vext16<MAX>(b), mc = vext16<MAX>(c), md = vext16<MAX>(d);
        const bool ha = cmp_holds<CMP>(ma, target), hb = cmp_holds<CMP>(mb, target);
        const bool hc = cmp_holds<CMP>(mc, target), hd = cmp_holds<CMP>(md, target);
        if (__any_sync(0xFFFFFFFFu, ha || hb || hc || hd)) {
            bal = __ballot_sync(0xFFFFFFFFu, ha);
            if (bal) { lm = ma; return Bk; }
            bal = __ballot_sync(0xFFFFFFFFu, hb);
            if (bal) { lm = mb; return Bk + BLK; }
            bal = __ballot_sync(0xFFFFFFFFu, hc);
            if (bal) { lm = mc; return Bk + 2 * BLK; }
            bal = __ballot_sync(0xFFFFFFFFu, hd);
            lm = md;
            return Bk + 3 * BLK;
        }
    }
    for (; Bk + 2 * BLK <= hi; Bk += 2 * BLK) {
        CNT(8);
        const uint4 a = *reinterpret_cast<const uint4 *>(sp + Bk + lane16);
        const uint4 b = *reinterpret_cast<const uint4 *>(sp + Bk + BLK + lane16);
        const uint32_t ma = vext16<MAX>(a), mb = vext16<MAX>(b);
        const bool ha = cmp_holds<CMP>(ma, target), hb = cmp_holds<CMP>(mb, target);
        if (__any_sync(0xFFFFFFFFu, ha || hb)) {
            bal = __ballot_sync(0xFFFFFFFFu, ha);
            if (bal) {
                lm = ma;
                return Bk;
            }
            bal = __ballot_sync(0xFFFFFFFFu, hb);
            lm = mb;
            return Bk + BLK;
        }
    }
    for (; Bk + BLK <= hi; Bk += BLK) {
        v = *reinterpret_cast<const uint4 *>(sp + Bk + lane16);
        lm = vext16<MAX>(v);
        bal = __ballot_sync(0xFFFFFFFFu, cmp_holds<CMP>(lm, target));
        if (bal) return Bk;
    }
    if (Bk < hi) {  // partial tail block
        CNT(10);
        lm = block_lane_ext<MAX>(sp, Bk, Bk, hi, has, v);
        bal = __ballot_sync(0xFFFFFFFFu, has && cmp_holds<CMP>(lm, target));
        if (bal) return Bk;
    }
    return -1;
}

// Range Scan locate: first stage offset in [lo, hi) inside lane L's 16 bytes of
// block Bk whose byte satisfies (byte CMP target); the lane is known to hold one.
template <int CMP>
__device__ __forceinline__ int stage_locate(const uint8_t *sp, int Bk, uint32_t bal, int lo, int hi,
                                            uint32_t target) {
    const int base = Bk + (__ffs(bal) - 1) * 16;
    const int j = lane_id() & 15;
    const int pos = base + j;
    const bool hit = lane_id() < 16 && pos >= lo && pos < hi && cmp_holds<CMP>(sp[pos], target);
    return base + __ffs(__ballot_sync(0xFFFFFFFFu, hit)) - 1;
}

// Saturating-byte masks (the sparse walk, the transfer tables).  Exact per-byte
// test for the saturating value: 0x80 marks each byte of x equal to 255 (MAX:
// (b & 0x7F) + 1 carries into bit 7 only for 0x7F, and b's own bit 7 must be
// set) or 0 (MIN: (b & 0x7F) + 0x7F | b has bit 7 clear only for 0); no carry
// crosses a byte.  One multiply gathers the four flags (bits 7, 15, 23, 31)
// into bits 28..31: flag k meets constant bit 21 - 7k, and every other partial
// product lands on a distinct bit below 28 or above 31.
template <bool MAX>
__device__ __forceinline__ uint32_t sat_nibble(uint32_t x) {
    const uint32_t f = MAX ? ((x & 0x7F7F7F7Fu) + 0x01010101u) & x & 0x80808080u
                           : ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
    return (f * 0x00204081u) >> 28;
}
// bit i set iff byte i of a lane's 16-byte vector is the saturating value
template <bool MAX>
__device__ __forceinline__ uint32_t sat_mask16(const uint4 &v) {
    return sat_nibble<MAX>(v.x) | (sat_nibble<MAX>(v.y) << 4) | (sat_nibble<MAX>(v.z) << 8) |
           (sat_nibble<MAX>(v.w) << 12);
}

// ---------------------------------------------------------------- chain engine
// run_chain walks the chunk chain of the stream fbase[0..Lf) that begins with
// a chunk at `start` (0 <= start < Lf).  Every boundary e < Lf (the start of
// the next chunk) is passed to emit.boundary(e), which returns true to stop
// the walk; when the chain's last chunk reaches Lf, emit.end() is called; when
// the bytes below read_end are exhausted first, emit.exhausted(c).  Bytes are
// read only below read_end.  All 32 lanes call this with identical arguments.
//
// yield_at (the sparse walk's partner, walk_chain): when non-null, the walk
// stops after YIELD_SAT consecutive saturated chunks (RAM: window maximum 0xFF;
// AE: an unbeaten saturating target) and stores the next chunk's start there
// (-1 otherwise), so that the sparse walk takes over again.
//
// Semantics are those of the oracle (oracle/cdc_oracle.c), with the chunk
// limit = min(Lf, s + max_size) (reading R5):
//   RAM:    M = max d[s, s+w); the chunk ends after the first i in [s+w, limit)
//           with d[i] >= M, else at limit; if s + w >= Lf it ends at Lf.
//   AE-Max: target t = s; while t + w < limit: if no byte of (t, t+w] exceeds
//           d[t] the chunk ends at t+w+1, else t = first byte of (t, t+w]
//           exceeding d[t]; once t + w >= limit it ends at limit.  (AE-Min:
//           "less" for "exceeds".)
//
// Inside a stage every position is an int offset from the stage's first byte
// (horizons beyond the stage clamp to FAR); the chain state between events is
// kept as 64-bit stream positions.  Between events the walker runs one of
// three tight loops: the RAM window's Extreme Byte Search (stage_window_max), a
// block-level Range Scan for the next event (stage_find_block), or -- for an
// AE target no byte can beat -- a direct jump to its deadline.
template <int ALGO, int STG = STAGE, class Emit>
__device__ void run_chain(const WarpRing &R, const uint8_t *__restrict__ fbase, int64_t Lf, int64_t start,
                          int64_t read_end, uint32_t w, uint64_t max_size, const L2Pol &pol, Emit &emit,
                          int64_t *yield_at = nullptr) {
    constexpr bool MAX = (ALGO != ALGO_AE_MIN);
    constexpr uint32_t SAT = MAX ? 255u : 0u;  // a target nothing can beat
    constexpr int FAR = 1 << 30;
    constexpr int CMP_BEAT = MAX ? CMP_GT : CMP_LT;
    const int lane = lane_id();
    if (read_end > Lf) read_end = Lf;
    const uint8_t *g0 = reinterpret_cast<const uint8_t *>(reinterpret_cast<uintptr_t>(fbase + start) &
                                                          ~static_cast<uintptr_t>(15));
    const int64_t B0 = g0 - fbase;
    const int64_t nbytes = ((read_end - B0) + 15) & ~static_cast<int64_t>(15);
    const int64_t nstages = (nbytes + STG - 1) / STG;

    if (lane == 0) {
        for (int i = 0; i < NST; ++i) mbar_init(&R.bar[i], 1);
        fence_barrier_init();
    }
    __syncwarp();

    int64_t issued = 0;
    auto issue = [&](int64_t k, int slot) {
        // operands computed by every lane (uniform, no divergent region); one elected lane issues
        const int64_t off = k * STG;
        const uint32_t bytes = (uint32_t)(nbytes - off < STG ? nbytes - off : STG);
        const uint64_t policy = B0 + off < pol.keep_until ? pol.keep : pol.stream;
        uint64_t *bar = &R.bar[slot];
        uint8_t *dst = R.buf + slot * STG;
        const uint8_t *src = g0 + off;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "elect.sync _|p, 0xffffffff;\n\t"
            "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
            "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%2], [%3], %1, [%0], %4;\n\t"
            "}" ::"r"(smem_addr(bar)), "r"(bytes), "r"(smem_addr(dst)), "l"(src), "l"(policy)
            : "memory");
    };
    for (; issued < nstages && issued < NST; ++issued) issue(issued, (int)issued);

    const int64_t W = (int64_t)w;
    const int W1 = w + 1 < (uint32_t)FAR ? (int)w + 1 : FAR;  // deadline distance t -> t+w+1, clamped
    // chain state (stream positions)
    int64_t s = start;                                                           // current chunk start
    int64_t limit = (Lf - s < (int64_t)max_size) ? Lf : s + (int64_t)max_size;  // chunk end bound
    int64_t c = s;                                                               // next byte to examine
    bool stop = false;
    bool scanning = false;  // RAM: false = window [s, s+w), true = scan for a byte >= M
    bool wsat = false;      // RAM: the window already holds a 255
    uint32_t M = 0, acc = 0;
    uint32_t ext = 0;       // AE: current target value
    int64_t t = 0;          // AE: current target position
    bool pending = true;    // AE: the chunk's first byte is the first target

    if constexpr (ALGO == ALGO_RAM) {
        if (s + W >= Lf) {  // window does not fit: a single final chunk
            emit.end();
            stop = true;
        }
    }

    if (yield_at) *yield_at = -1;
    int sat_run = 0;        // consecutive saturated chunks (yield_at)
    bool last_sat = false;  // the chunk ending at the next boundary is saturated
    // a boundary at e: returns true when the walk stops
    auto on_boundary = [&](int64_t e) -> bool {
        if (e >= Lf) {
            emit.end();
            return true;
        }
        if (emit.boundary(e)) return true;
        if (yield_at) {
            sat_run = last_sat ? sat_run + 1 : 0;
            if (sat_run >= YIELD_SAT && e + (int64_t)w < Lf) {
                *yield_at = e;  // the sparse walk continues with the chunk at e
                return true;
            }
        }
        s = e;
        c = e;
        limit = (Lf - s < (int64_t)max_size) ? Lf : s + (int64_t)max_size;
        if constexpr (ALGO == ALGO_RAM) {
            scanning = false;
            wsat = false;
            acc = 0;
            if (s + W >= Lf) {
                emit.end();
                return true;
            }
        } else {
            pending = true;
        }
        return false;
    };

    int slot = 0;
    uint32_t parity = 0;
    int64_t k = 0;
    ET_DECL
    ET_BEGIN(et_t1);
    for (; k < nstages && !stop; ++k) {
        CNT(0);
        const int64_t SB = B0 + k * STG;
        mbar_wait(&R.bar[slot], parity);
        const uint8_t *sp = R.buf + slot * STG;
        auto rel = [&](int64_t x) -> int {  // x >= SB
            const int64_t d = x - SB;
            return d > FAR ? FAR : (int)d;
        };
        const int endr = rel(read_end) < STG ? rel(read_end) : STG;
        int cr = (int)(c - SB);
        int limr = rel(limit);
        // RAM: window end s+w while not scanning; AE: target deadline t+w+1
        int hor = FAR;
        if constexpr (ALGO == ALGO_RAM) {
            if (!scanning) hor = rel(s + W);
        } else {
            if (!pending) hor = rel(t + W + 1);
        }
        // a boundary at stage offset er
        auto event = [&](int er) -> bool {
            CNT(6);
            if (on_boundary(SB + er)) return true;
            cr = er;
            limr = rel(limit);
            if constexpr (ALGO == ALGO_RAM) hor = rel(s + W);
            else hor = FAR;
            return false;
        };
        ET_HALO_STAGE(emit.in_halo(), et_t1);
        ET_ADD(0, et_t1);  // stage transition: wait + setup
        while (cr < endr) {
            ET_VAR(eit)
            ET_BEGIN(eit);
            if constexpr (ALGO == ALGO_RAM) {
                if (!scanning) {
                    const int hi = hor < endr ? hor : endr;
                    CNT(11);
                    if (!wsat) wsat = stage_window_max(sp, cr, hi, acc);  // a saturated window skips its rest
                    cr = hi;
                    if (cr == hor) {
                        M = wsat ? 255u : warp_ext<true>(acc);
                        last_sat = M == 255u;
                        scanning = true;
                        hor = FAR;
                    }
                } else {
                    const int hi = limr < endr ? limr : endr;
                    uint32_t bal = 0, lm;
                    bool has;
                    CNT(12);
                    const int Bk = stage_find_block<CMP_GEQ>(sp, cr, hi, M, bal, lm, has);
                    int er;
                    if (Bk >= 0) {
                        er = stage_locate<CMP_GEQ>(sp, Bk, bal, cr, hi, M) + 1;  // boundary byte ends the chunk
                    } else {
                        cr = hi;
                        if (cr != limr) break;
                        er = limr;  // cap or end of stream
                    }
                    if (event(er)) {
                        stop = true;
                        break;
                    }
                }
            } else {
                // pending: the chunk's first byte is its first target, deadline s + w + 1
                if (pending) {
                    t = SB + cr;
                    hor = cr + W1 < FAR ? cr + W1 : FAR;
                }
                int hi = hor < limr ? hor : limr;
                hi = hi < endr ? hi : endr;
                if (ext == SAT && !pending) CNT(5);
                const bool sat_iter = ext == SAT && !pending;
                (void)sat_iter;
                int Bk = -1;  // first block of [cr, hi) that can hold the next target
                uint32_t lm = 0;
                bool has = false;
                if (pending) {
                    // Every byte of [s, hi) lies in the window of the first target s,
                    // so the collapse below applies from the chunk's first byte on: the
                    // target after [s, hi) is the first occurrence of its extreme (no
                    // separate first-byte step and record scan).
                    CNT(1);
                    Bk = cr & ~(BLK - 1);
                    uint4 v0;
                    lm = block_lane_ext<MAX>(sp, Bk, cr, hi < Bk + BLK ? hi : Bk + BLK, has, v0);
                    pending = false;
                } else if (ext != SAT && cr < hi) {
                    uint32_t bal = 0;
                    CNT(2);
                    ET_VAR(e1)
                    ET_BEGIN(e1);
                    Bk = stage_find_block<CMP_BEAT>(sp, cr, hi, ext, bal, lm, has);
                    ET_ADD(1, e1);
                }
                if (Bk >= 0) {
                    CNT(3);
                    ET_VAR(e2)
                    ET_BEGIN(e2);
                    // Every byte of [cr, hi) lies inside the current target's window
                    // (hi <= t + w + 1), so the records of [cr, hi) follow one another
                    // within w bytes and none ends the chunk: the last of them -- the
                    // first occurrence of the range's extreme -- is the new target.
                    // One Extreme Byte Search (§4.1) over the rest of the range (it
                    // stops at the first block holding the saturating value) replaces
                    // a record event per block.
                    const int lo = cr > Bk ? cr : Bk;
                    uint32_t lacc = has ? lm : neutral<MAX>();
                    int lblk = Bk, Bs = -1;
                    if (__any_sync(0xFFFFFFFFu, has && lm == SAT)) Bs = Bk;
                    int B = Bk + BLK;
                    for (; Bs < 0 && B + 2 * BLK <= hi; B += 2 * BLK) {  // two blocks in flight
                        const uint32_t m0 = vext16<MAX>(*reinterpret_cast<const uint4 *>(sp + B + lane * 16));
                        const uint32_t m1 = vext16<MAX>(*reinterpret_cast<const uint4 *>(sp + B + BLK + lane * 16));
                        if (beats<MAX>(m0, lacc)) {
                            lacc = m0;
                            lblk = B;
                        }
                        if (beats<MAX>(m1, lacc)) {
                            lacc = m1;
                            lblk = B + BLK;
                        }
                        const uint32_t s0 = __ballot_sync(0xFFFFFFFFu, m0 == SAT);
                        const uint32_t s1 = __ballot_sync(0xFFFFFFFFu, m1 == SAT);
                        if (s0 | s1) Bs = s0 ? B : B + BLK;
                    }
                    for (; Bs < 0 && B < hi; B += BLK) {
                        uint32_t mb;
                        if (B + BLK <= hi) {
                            mb = vext16<MAX>(*reinterpret_cast<const uint4 *>(sp + B + lane * 16));
                        } else {
                            bool h2;
                            uint4 v2;
                            mb = block_lane_ext<MAX>(sp, B, B, hi, h2, v2);
                        }
                        if (beats<MAX>(mb, lacc)) {
                            lacc = mb;
                            lblk = B;
                        }
                        if (__any_sync(0xFFFFFFFFu, mb == SAT)) Bs = B;
                    }
                    const uint32_t m = Bs >= 0 ? SAT : warp_ext<MAX>(lacc);
                    const int Bf = Bs >= 0 ? Bs : (int)__reduce_min_sync(0xFFFFFFFFu, lacc == m ? (uint32_t)lblk : 0x7FFFFFFFu);
                    const int flo = lo > Bf ? lo : Bf, fhi = hi < Bf + BLK ? hi : Bf + BLK;
                    bool hf;
                    uint4 vf;
                    const uint32_t lmf = block_lane_ext<MAX>(sp, Bf, flo, fhi, hf, vf);
                    const uint32_t b2 = __ballot_sync(0xFFFFFFFFu, hf && lmf == m);
                    const int r = stage_locate<CMP_EQ>(sp, Bf, b2, flo, fhi, m);
                    ext = m;
                    cr = Bs >= 0 ? fhi : hi;  // nothing in (r, cr) beats m
                    t = SB + r;
                    hor = r + W1 < FAR ? r + W1 : FAR;
                    ET_ADD(2, e2);
                    continue;
                }
                cr = hi;
#ifdef CDC_EVTIME
                if (sat_iter) { ET_ADD(5, eit); } else { ET_ADD(6, eit); }
#endif
                int er;
                if (cr == hor && hor <= limr) er = hor;  // target unbeaten over its window
                else if (cr == limr) er = limr;         // cap or end of stream
                else break;                             // stage exhausted
                last_sat = er == hor && ext == SAT;
                ET_VAR(e3)
                ET_BEGIN(e3);
                if (event(er)) {
                    stop = true;
                    break;
                }
                ET_ADD(3, e3);
            }
        }
        c = SB + cr;
        ET_BEGIN(et_t1);
        __syncwarp();
        if (!stop && issued < nstages) {  // refill this slot with stage k + NST
            issue(issued, slot);
            ++issued;
        }
        if (++slot == NST) {
            slot = 0;
            parity ^= 1u;
        }
    }
    // all bytes below read_end consumed without the emitter stopping
    if (!stop) {
        if (c >= Lf) emit.end();
        else emit.exhausted(c);
    }
    ET_FLUSH
    // drain copies still in flight (stages k .. issued-1) before the ring is reused or the CTA exits
    for (; k < issued; ++k) {
        mbar_wait(&R.bar[slot], parity);
        if (++slot == NST) {
            slot = 0;
            parity ^= 1u;
        }
    }
    __syncwarp();
    if (lane == 0) {
        for (int i = 0; i < NST; ++i) mbar_inval(&R.bar[i]);  // the ring may be re-initialised by the caller
        R.bar[FETCH_SLOT] += (uint64_t)(issued * STG < nbytes ? issued * STG : nbytes);
    }
    __syncwarp();
}

// ---------------------------------------------------------------- sparse walker
// Saturated chunks need only a few bytes ("sparse walk"):
//   RAM (§2.1.2 l.198): a window [s, s+w) that holds 0xFF has maximum 0xFF, so
//     the chunk ends after the first 0xFF in [s+w, limit), else at limit -- the
//     rest of the window is never needed;
//   AE-Max (l.169; AE-Min with 0x00): if the first saturating byte q of
//     [s, s+w] exists, every earlier target is beaten within w bytes (q is at
//     most w after it) and nothing beats q, so the chunk ends at q+w+1 (at
//     limit when q+w >= limit); when s+w >= limit it ends at limit whatever
//     the bytes.
// A chunk's *decisive bytes* start at x = s+w (RAM) or x = s (AE).  Every
// chunk but a stream's last is longer than w, so the decisive bytes of the
// k-th chunk after this one start at or after s + GAP + (k-1)(w+1), GAP =
// 2w+1 (RAM) or w+1 (AE).  At the start of each chunk the walker already
// issues a bulk copy (TMA, into its idle ring) of the SP_SPEC bytes from there
// for k = SP_DEPTH: those chunks' decisive bytes, unless the waits for a
// saturating byte of the chunks up to it add up to more than SP_SPEC.  With
// SP_DEPTH copies in flight behind the one being waited for, a chunk costs
// 1/(SP_DEPTH+1) of a memory round trip, and only ~SP_SPEC bytes per chunk are
// read.  A scan that runs past its region continues with copies of SP_SPEC
// bytes into the continuation slots;
// RAM's window test looks at the bytes after the last boundary (still in the
// slot that held it), then probes the window.  At the first chunk that cannot
// be decided this way it stops and returns false with the chunk's start in
// `resume` (the caller continues with run_chain from there).  Returns true
// when the walk ended (emitter stop, stream end, exhaustion) with the emitter
// calls run_chain would have made.
#ifndef CDC_SP_SPEC
#define CDC_SP_SPEC 2048
#endif
constexpr int SP_SPEC = CDC_SP_SPEC;  // bytes per speculative or continuation copy (multiple of 16, <= SP_SLOT)
#ifndef CDC_SP_SLOT
#define CDC_SP_SLOT 2048
#endif
constexpr int SP_SLOT = CDC_SP_SLOT;  // slot stride in the ring
// Speculative copies in flight: at the start of chunk n the walker issues the
// copy for chunk n + SP_DEPTH (whose decisive bytes start at or after
// s + GAP + (SP_DEPTH - 1)(w + 1): every chunk is longer than w), so a chunk
// costs ~1/(SP_DEPTH + 1) of a memory round trip while the overshoots of
// SP_DEPTH + 1 chunks add up to less than SP_SPEC.  Measured: a
// lone walker waits only ~105 of its ~1,400 cycles per chunk for the copy, and
// SP_DEPTH 2 is slower everywhere (configs[3] 1.20 -> 1.28 ms), so 1 it is.
#ifndef CDC_SP_DEPTH
#define CDC_SP_DEPTH 1
#endif
constexpr int SP_DEPTH = CDC_SP_DEPTH;
static_assert(SP_DEPTH == 1 || SP_DEPTH == 2, "SP_DEPTH");
constexpr int SP_CS0 = SP_DEPTH + 1;      // slots 0..SP_DEPTH rotate per chunk (speculative regions);
constexpr int SP_NSLOT = SP_DEPTH + 3;    // SP_CS0, SP_CS0 + 1: continuation regions (ping-pong)
static_assert(SP_NSLOT <= FETCH_SLOT, "one mbarrier per sparse-walk slot before the fetch counter");
static_assert(Ring<5120>::BYTES >= SP_NSLOT * SP_SLOT, "sparse walk needs SP_NSLOT slots in every ring (stages of >= 5 KiB)");
static_assert(SP_SPEC % 16 == 0 && SP_SPEC <= SP_SLOT, "SP_SPEC");

// First saturating byte in [lo, hi) among the slot's bytes [P, P + n) (file
// positions), or -1: one 512-byte block per step, exact per-byte masks
// (sat_mask16), one ballot per block.
// (more: set when the same block holds another such byte in (result, hi))
template <bool MAX, typename IX = int64_t>
__device__ __forceinline__ IX sm_first(const uint8_t *sp, IX P, int n, IX lo, IX hi, bool *more = nullptr) {
    if (lo < P) lo = P;
    if (hi > P + n) hi = P + n;
    if (lo >= hi) return IX(-1);
    const int a = (int)(lo - P), b = (int)(hi - P);
    const int l16 = lane_id() * 16;
    for (int B = a & ~(BLK - 1); B < b; B += BLK) {
        const uint4 v = *reinterpret_cast<const uint4 *>(sp + B + l16);
        const int q = B + l16;
        const int ka = min(max(a - q, 0), 16), kb = min(max(b - q, 0), 16);
        const uint32_t m = sat_mask16<MAX>(v) & ((1u << kb) - 1u) & ~((1u << ka) - 1u);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m != 0u);
        if (bal) {
            const int L = __ffs(bal) - 1;
            const uint32_t mL = __shfl_sync(0xFFFFFFFFu, m, L);
            if (more) *more = (mL & (mL - 1u)) != 0u || (bal >> L) > 1u;
            return P + (IX)(B + 16 * L + (__ffs(mL) - 1));
        }
    }
    return IX(-1);
}
// sm_first on a 32-bit shared-window address sp, the lane's byte offset l16 =
// 16 * lane passed in (the sparse walk keeps both in registers)
template <bool MAX, typename IX>
__device__ __forceinline__ IX sm_first_s(uint32_t sp, int l16, IX P, int n, IX lo, IX hi, bool *more = nullptr) {
    if (lo < P) lo = P;
    if (hi > P + n) hi = P + n;
    if (lo >= hi) return IX(-1);
    const int a = (int)(lo - P), b = (int)(hi - P);
    for (int B = a & ~(BLK - 1); B < b; B += BLK) {
        const uint4 v = lds128(sp + (uint32_t)(B + l16));
        const int q = B + l16;
        const int ka = min(max(a - q, 0), 16), kb = min(max(b - q, 0), 16);
        const uint32_t m = sat_mask16<MAX>(v) & ((1u << kb) - 1u) & ~((1u << ka) - 1u);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m != 0u);
        if (bal) {
            const int L = __ffs(bal) - 1;
            const uint32_t mL = __shfl_sync(0xFFFFFFFFu, m, L);
            if (more) *more = (mL & (mL - 1u)) != 0u || (bal >> L) > 1u;
            return P + (IX)(B + 16 * L + (__ffs(mL) - 1));
        }
    }
    return IX(-1);
}
#ifndef CDC_SP_FIND
#define CDC_SP_FIND 0
#endif
template <int CMP, typename IX = int64_t>
__device__ __forceinline__ IX sm_find(const uint8_t *sp, IX P, int n, IX lo, IX hi, uint32_t target);
// the sparse walk's region search for the saturating value (CDC_SP_FIND: 0 =
// sm_first, 1 = the ring walker's Range Scan)
template <bool MAX, typename IX = int64_t>
__device__ __forceinline__ IX sm_sat(const uint8_t *sp, IX P, int n, IX lo, IX hi) {
    if (CDC_SP_FIND == 0) return sm_first<MAX, IX>(sp, P, n, lo, hi);
    return sm_find<MAX ? CMP_GEQ : CMP_LEQ, IX>(sp, P, n, lo, hi, MAX ? 255u : 0u);
}

// First byte of the slot's region [P, P + n) (file positions) in [lo, hi) that
// satisfies (byte CMP target), or -1: the ring walker's block-level Range Scan
// (stage_find_block: a per-lane extreme over 16-byte vectors, four blocks in
// flight, one ballot per block) and its in-lane locate.
template <int CMP, typename IX>
__device__ __forceinline__ IX sm_find(const uint8_t *sp, IX P, int n, IX lo, IX hi, uint32_t target) {
    if (lo < P) lo = P;
    if (hi > P + n) hi = P + n;
    if (lo >= hi) return IX(-1);
    const int a = (int)(lo - P), b = (int)(hi - P);
    uint32_t bal = 0, lm = 0;
    bool has = false;
    const int Bk = stage_find_block<CMP>(sp, a, b, target, bal, lm, has);
    if (Bk < 0) return IX(-1);
    return P + (IX)stage_locate<CMP>(sp, Bk, bal, a, b, target);
}

#ifdef CDC_SPTIME  // diagnostic: sparse walk cycle accounting into g_evt[11..15] (tools/sparse_probe.py)
#define SPT_DECL long long spt_acc[5] = {0, 0, 0, 0, 0}, spt_t = 0, spt_0 = clock64();
#define SPT_BEGIN spt_t = clock64()
#define SPT_ADD(i) spt_acc[i] += clock64() - spt_t
#define SPT_FLUSH                                                                       \
    if (lane == 0) {                                                                    \
        spt_acc[4] = clock64() - spt_0;                                                 \
        for (int q = 0; q < 5; ++q) atomicAdd(&g_evt[11 + q], (unsigned long long)spt_acc[q]); \
    }
#else
#define SPT_DECL
#define SPT_BEGIN
#define SPT_ADD(i)
#define SPT_FLUSH
#endif
// IX: the type of positions inside the walk, relative to its start (int when
// the rest of the file and max_size fit in 2^29 -- every batch file of
// configs[3] --, which halves the bookkeeping instructions of a chunk;
// int64_t otherwise).
template <int ALGO, typename IX, class Emit>
__device__ bool sparse_chain(const WarpRing &R, const uint8_t *__restrict__ fbase0, int64_t Lf0, int64_t org,
                             int64_t read_end0, uint32_t w, uint64_t max_size0, Emit &emit, int64_t &resume) {
    constexpr bool MAX = (ALGO != ALGO_AE_MIN);
    constexpr bool RAM = (ALGO == ALGO_RAM);
    const int lane = lane_id();
    const IX W = (IX)w;
    const uint8_t *__restrict__ fbase = fbase0 + org;  // positions below are relative to org
    // (the int instance clamps a distant file end to 2^30: every position it forms stays
    // below that, so every comparison with the file end comes out as with the real one)
    const IX Lf = (IX)(sizeof(IX) == 4 && Lf0 - org > (1ll << 30) ? (1ll << 30) : Lf0 - org);
    const IX max_size = (IX)max_size0;
    const IX read_end = (IX)((read_end0 < Lf0 ? read_end0 : Lf0) - org);
    const uint64_t pol = l2_evict_first_policy();
    if (lane == 0) {
        for (int i = 0; i < SP_NSLOT; ++i) mbar_init(&R.bar[i], 1);
        fence_barrier_init();
    }
    __syncwarp();
    // shared-window addresses of the slots and their mbarriers, and the lane's byte
    // offset, kept in registers (opaque: not rebuilt from the thread index per use)
    uint32_t sbuf = smem_addr(R.buf), sbar = smem_addr(R.bar);
    int l16 = lane * 16;
    asm volatile("" : "+r"(sbuf), "+r"(sbar), "+r"(l16));
    auto find = [&](int slot, IX P, int n, IX lo, IX hi, bool *more) -> IX {
        if (CDC_SP_FIND == 0) return sm_first_s<MAX, IX>(sbuf + slot * SP_SLOT, l16, P, n, lo, hi, more);
        return sm_sat<MAX, IX>(R.buf + slot * SP_SLOT, P, n, lo, hi);
    };
    auto find_ff = [&](int slot, IX P, int n, IX lo, IX hi) -> IX {  // RAM's window test: a 0xFF
        if (CDC_SP_FIND == 0) return sm_first_s<true, IX>(sbuf + slot * SP_SLOT, l16, P, n, lo, hi);
        return sm_sat<true, IX>(R.buf + slot * SP_SLOT, P, n, lo, hi);
    };
    uint32_t pend = 0, par = 0;  // per slot: copy in flight; parity of its next completion
    uint32_t fetched = 0;        // bytes copied by this call (flushed into R.bar[FETCH_SLOT] at the end)
    // copy of the bytes from x (rounded down to 16 B, at most nb bytes, not past the
    // granule holding byte Lf - 1) into slot `slot`; P, N: the region's start and size
    auto issue = [&](int slot, IX x, int nb, IX &P, int &N) {
        P = x - (IX)(reinterpret_cast<uintptr_t>(fbase + x) & 15u);
        const IX avail = ((Lf - P) + 15) & ~static_cast<IX>(15);
        N = (int)(avail < (IX)nb ? (avail > 0 ? avail : 0) : (IX)nb);
        if (N > 0) {
            fetched += (uint32_t)N;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "elect.sync _|p, 0xffffffff;\n\t"
                "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
                "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%2], [%3], %1, [%0], %4;\n\t"
                "}" ::"r"(sbar + 8 * slot), "r"((uint32_t)N), "r"(sbuf + slot * SP_SLOT), "l"(fbase + P),
                "l"(pol)
                : "memory");
            pend |= 1u << slot;
        }
    };
    auto wait = [&](int slot) {
        if ((pend >> slot) & 1u) {
            mbar_wait_s(sbar + 8 * slot, (par >> slot) & 1u);
            par ^= 1u << slot;
            pend &= ~(1u << slot);
        }
    };
    // Continuation regions (a stretch without a saturating byte: the rest of a
    // chunk past its speculative copy, or RAM's window probes) alternate between
    // slots 2 and 3.  From the second region of a run on, the region after the
    // one to be scanned is copied into the other slot first, so two copies are
    // in flight and a long stretch (a zero-filled region) costs half a round
    // trip per region instead of one.  cont() returns the slot holding the
    // region that starts at x (its [Pc, Pc + Nc)); cs, pf, pfP, pfN, run: the
    // run's state (the next slot, the slot and region of a copy issued ahead).
    auto cont = [&](IX x, IX hi, int &cs, int &pf, IX &pfP, int &pfN, bool &run, IX &Pc, int &Nc) -> int {
        int s_;
        if (pf >= 0 && pfP == x) {
            s_ = pf;
            Pc = pfP;
            Nc = pfN;
        } else {
            s_ = cs;
            wait(s_);
            issue(s_, x, SP_SPEC, Pc, Nc);
        }
        pf = -1;
        if (run && Nc > 0 && Pc + Nc < hi) {
            const int o = s_ == SP_CS0 ? SP_CS0 + 1 : SP_CS0;
            wait(o);
            issue(o, Pc + Nc, SP_SPEC, pfP, pfN);
            pf = o;
        }
        run = true;
        cs = s_ == SP_CS0 ? SP_CS0 + 1 : SP_CS0;
        wait(s_);
        return s_;
    };
    SPT_DECL
    auto finish = [&](bool r) -> bool {
        SPT_FLUSH
        for (int i = 0; i < SP_NSLOT; ++i) wait(i);
        __syncwarp();
        if (lane == 0) {
            for (int i = 0; i < SP_NSLOT; ++i) mbar_inval(&R.bar[i]);
            R.bar[FETCH_SLOT] += fetched;
        }
        __syncwarp();
        return r;
    };
    const IX GAP = RAM ? 2 * W + 1 : W + 1;  // the next chunk's decisive bytes start at or after s + GAP
    IX s = 0;
    const IX GAP2 = GAP + W + 1;  // (SP_DEPTH 2) ... and those of the chunk after it at or after s + GAP2
    int cur = 0;        // slot of this chunk's speculative region (slots 0..SP_DEPTH in rotation)
    IX cP = 0;          // ... its region [cP, cP + cN)
    int cN = 0;
    [[maybe_unused]] int n1 = 1, n2 = 2; // (SP_DEPTH 2) slots of the next chunk's region [aP, aP + aN) and of the one after it
    [[maybe_unused]] IX aP = 0;
    [[maybe_unused]] int aN = 0;
    int rs = -1;        // RAM: slot holding the bytes right after s, its region [rP, rP + rN)
    IX rP = 0;
    int rN = 0;
    IX P2 = 0;          // the continuation slots' current region
    int N2 = 0;
    bool wsat = false;  // RAM: this chunk's window is known to hold a 0xFF
    for (;;) {
        if (RAM && s + W >= Lf) {  // the window does not fit: a single final chunk
            emit.end();
            return finish(true);
        }
        const IX limit = (Lf - s < max_size) ? Lf : s + max_size;
        SPT_BEGIN;
        if (RAM && !wsat) {  // does the window [s, s+w) hold a 0xFF?
            const IX wend = s + W < read_end ? s + W : read_end;
            bool sat = false;
            IX x = s;
            if (rs >= 0) {
                sat = find_ff(rs, rP, rN, s, wend) >= 0;
                if (rP + rN > x) x = rP + rN;
            }
            int cs = SP_CS0, pf = -1, pfN = 0;
            IX pfP = 0;
            bool run = false;
            while (!sat && x < wend) {
                CNT(15);
                const int s2 = cont(x, wend, cs, pf, pfP, pfN, run, P2, N2);
                if (N2 <= 0) break;
                sat = find_ff(s2, P2, N2, x, wend) >= 0;
                x = P2 + N2;
            }
            if (!sat) {  // the ring walker decides this chunk
                resume = org + s;
                return finish(false);
            }
        }
        SPT_ADD(0);
        const int nxt = SP_DEPTH == 1 ? (cur ^ 1) : n2;
        IX nP = 0;
        int nN = 0;
        wait(nxt);  // (the last chunk's region, already consumed)
        if constexpr (SP_DEPTH == 1) {
            if (s + GAP < Lf) issue(nxt, s + GAP, SP_SPEC, nP, nN);
        } else {
            if (aN <= 0 && s + GAP < Lf) issue(n1, s + GAP, SP_SPEC, aP, aN);  // (the walk's first chunk)
            if (s + GAP2 < Lf) issue(nxt, s + GAP2, SP_SPEC, nP, nN);
        }
        IX e;
        if (!RAM && s + W >= limit) {
            e = limit;  // no target's window fits before the limit
        } else {
            const IX x0 = RAM ? s + W : s;
            const IX hi = RAM ? (limit < read_end ? limit : read_end) : s + W + 1;
            if (!RAM && hi > read_end) {
                resume = org + s;
                return finish(false);
            }
            if (!(cN > 0 && cP <= x0 && x0 < cP + cN)) {  // not covered by the speculative copy
                CNT(13);
                wait(cur);
                issue(cur, x0, SP_SPEC, cP, cN);
            }
            SPT_BEGIN;
            wait(cur);
            SPT_ADD(1);
            SPT_BEGIN;
            int slot = cur;
            IX P = cP;
            int N = cN;
            bool more = false;  // (RAM: another 0xFF within 512 bytes after the boundary byte)
            IX pos = find(cur, cP, cN, x0, hi, &more);
            int cs = SP_CS0, pf = -1, pfN = 0;
            IX pfP = 0;
            bool run = false;
            while (pos < 0 && P + N < hi && N > 0) {  // continue past the region
                const IX x = P + N > x0 ? P + N : x0;
                CNT(14);
                slot = cont(x, hi, cs, pf, pfP, pfN, run, P2, N2);
                P = P2;
                N = N2;
                pos = find(slot, P2, N2, x, hi, &more);
            }
            if (RAM) {
                if (pos >= 0) {
                    e = pos + 1;
                } else if (hi == limit) {
                    e = limit;  // cap or end of stream
                } else {
                    emit.exhausted(org + read_end);
                    return finish(true);
                }
                rs = slot;
                rP = P;
                rN = N;
                wsat = pos >= 0 && more;  // the next window [e, e + w) holds that 0xFF (w >= 512)
            } else {
                if (pos < 0) {  // no saturating byte in [s, s+w]: the ring walker decides this chunk
                    resume = org + s;
                    return finish(false);
                }
                e = pos + W < limit ? pos + W + 1 : limit;
            }
            SPT_ADD(2);
        }
        if (e >= Lf) {
            emit.end();
            return finish(true);
        }
        SPT_BEGIN;
        const bool stop_ = emit.boundary(org + e);
        SPT_ADD(3);
        if (stop_) return finish(true);
        s = e;
        if constexpr (SP_DEPTH == 1) {
            cur = nxt;
            cP = nP;
            cN = nN;
        } else {
            n2 = cur;  // consumed: the next chunk's copy goes there
            cur = n1;
            cP = aP;
            cN = aN;
            n1 = nxt;
            aP = nP;
            aN = nN;
        }
    }
}

// The walk of a chain from a chunk start: sparse while the chunks saturate,
// the TMA-ring walker from the first chunk the sparse walk cannot decide, and
// back to the sparse walk after YIELD_SAT saturated chunks in a row.
// SPM: which sparse walks the kernel carries -- 0 none (its launches never set
// `sparse`; configs[1]'s window is below the sparse walk's minimum, and without
// that code its walker keeps fewer registers), 1 the int64-position instance,
// 2 also the int-position instance, taken when the walk's byte range and
// max_size are below 2^28 (every walk of a batch, of K-phase and of a
// single-stream segment of a few hundred MB).
template <int ALGO, int STG = STAGE, int SPM = 1, class Emit>
__device__ __forceinline__ void walk_chain(bool sparse, const WarpRing &R, const uint8_t *__restrict__ fbase, int64_t Lf,
                                           int64_t start, int64_t read_end, uint32_t w, uint64_t max_size,
                                           const L2Pol &pol, Emit &emit) {
    if constexpr (SPM == 0) {
        run_chain<ALGO, STG>(R, fbase, Lf, start, read_end, w, max_size, pol, emit);
        return;
    }
    if (!sparse) {
        run_chain<ALGO, STG>(R, fbase, Lf, start, read_end, w, max_size, pol, emit);
        return;
    }
    if constexpr (SPM != 0) for (;;) {
        int64_t resume = start;
        // (int positions: read_end - start and max_size below 2^28 keep every position the
        // walk forms below 2^30; the file end is clamped to 2^30 beyond that)
        const bool narrow = SPM == 2 && read_end - start < (1ll << 28) && max_size < (1ull << 28);
        bool done;
        if constexpr (SPM == 2)
            done = narrow ? sparse_chain<ALGO, int>(R, fbase, Lf, start, read_end, w, max_size, emit, resume)
                          : sparse_chain<ALGO, int64_t>(R, fbase, Lf, start, read_end, w, max_size, emit, resume);
        else
            done = sparse_chain<ALGO, int64_t>(R, fbase, Lf, start, read_end, w, max_size, emit, resume);
        if (done) return;
        int64_t y = -1;
        run_chain<ALGO, STG>(R, fbase, Lf, resume, read_end, w, max_size, pol, emit, &y);
        if (y < 0) return;
        start = y;
    }
}

}  // namespace cdc
