// cdc_device.cuh -- device building blocks of the sm_100a chunker.
//
//  * PTX wrappers: mbarrier, 1-D TMA bulk copy (cp.async.bulk -> UBLKCP),
//    L2 evict-first policy, acquire/release flags.
//  * Byte SIMD: Extreme Byte Search (§4.1) as a per-lane max/min tree
//    over 16-byte vectors using the native DPX VIMNMX3.U16x2 instruction and
//    a CREDUX warp reduction; Range Scan (§4.2) as per-byte compare masks
//    collapsed to one bit per byte, a warp ballot and __ffs -- the GPU form of
//    the paper's VCMP + VMASK "packed scanning".
//  * run_chain: one warp walks the chunk chain of one stream from a given
//    start, streaming the bytes through a private shared-memory ring of
//    NST 2 KiB stages filled by TMA, and reports every chunk boundary to an
//    Emit policy.  RAM (§2.1.2 l.198; §4.3 l.355) and AE-Max/AE-Min (§2.1.2
//    l.169-171; §4.3 l.357-359) are written as single-pass state machines
//    that consume each byte once.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cdc {

constexpr int STAGE = 2048;            // bytes per TMA stage = one warp step (4 x 512 B)
constexpr int NST = 8;                 // ring depth per warp (16 KiB)
constexpr int RING_BYTES = STAGE * NST;
constexpr int RING_SMEM = RING_BYTES + NST * 8;

enum { ALGO_RAM = 0, ALGO_AE_MAX = 1, ALGO_AE_MIN = 2 };
enum { CMP_GT = 0, CMP_GEQ = 1, CMP_LT = 2, CMP_LEQ = 3, CMP_EQ = 4 };

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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
__device__ unsigned long long *g_dbg_fwd = nullptr;  // set with g_dbg (debug only)
// Watchdog: a stage that has not landed within ~10 s (clock64) means a lost
// bulk copy; record the raw barrier word and trap instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const long long t0 = clock64();
    bool noted = false;
    while (!mbar_try_wait(bar, parity)) {
        const long long dt = clock64() - t0;
        if (!noted && dt > 2000000000ll) {
            noted = true;
            unsigned long long *p = g_dbg_fwd;
            if (p) {
                unsigned long long v;
                asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(smem_addr(bar)));
                volatile unsigned long long *q = p + (8191ull * 4);
                q[0] = 0xBADull; q[1] = v; q[2] = parity; q[3] = ((unsigned long long)blockIdx.x << 32) | threadIdx.x;
            }
        }
        if (dt > 20000000000ll) __trap();
    }
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// 1-D bulk copy global -> shared, completion signalled on an mbarrier (TMA; SASS UBLKCP).
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------- byte SIMD
// Max/min of bytes with the DPX 3-input u16x2 min/max: a raw word's 16-bit
// halves carry bytes 1 and 3 in their high bytes; the word shifted left by 8
// carries bytes 0 and 2 there.  The high byte of the u16 extreme of a set of
// halves is the extreme of their high bytes, whatever the low bytes are.
template <bool MAX>
__device__ __forceinline__ uint32_t ext3(uint32_t a, uint32_t b, uint32_t c) {
    if constexpr (MAX)
        return __vimax3_u16x2(a, b, c);
    else
        return __vimin3_u16x2(a, b, c);
}
template <bool MAX>
__device__ __forceinline__ void acc16(const uint4 &v, uint32_t &hi, uint32_t &lo) {
    hi = ext3<MAX>(hi, v.x, v.y);
    hi = ext3<MAX>(hi, v.z, v.w);
    lo = ext3<MAX>(lo, v.x << 8, v.y << 8);
    lo = ext3<MAX>(lo, v.z << 8, v.w << 8);
}
template <bool MAX>
__device__ __forceinline__ uint32_t acc_init() {
    return MAX ? 0u : 0xFFFFFFFFu;
}
// the extreme byte held by a (hi, lo) accumulator pair
template <bool MAX>
__device__ __forceinline__ uint32_t acc_extreme(uint32_t hi, uint32_t lo) {
    uint32_t m = ext3<MAX>(hi, lo, acc_init<MAX>());
    uint32_t a = m >> 24, b = (m >> 8) & 0xFFu;
    return MAX ? max(a, b) : min(a, b);
}
template <bool MAX>
__device__ __forceinline__ uint32_t warp_extreme(uint32_t v) {
    if constexpr (MAX)
        return __reduce_max_sync(0xFFFFFFFFu, v);
    else
        return __reduce_min_sync(0xFFFFFFFFu, v);
}

// per-byte comparison (0xFF where true) of 4 packed bytes against a broadcast target
template <int CMP>
__device__ __forceinline__ uint32_t vcmp4(uint32_t x, uint32_t t4) {
    if constexpr (CMP == CMP_GT) return __vcmpgtu4(x, t4);
    else if constexpr (CMP == CMP_GEQ) return __vcmpgeu4(x, t4);
    else if constexpr (CMP == CMP_LT) return __vcmpltu4(x, t4);
    else if constexpr (CMP == CMP_LEQ) return __vcmpleu4(x, t4);
    else return __vcmpeq4(x, t4);
}
// 0xFF/0x00 bytes -> 4 bits (byte i -> bit i)
__device__ __forceinline__ uint32_t pack4(uint32_t m) { return ((m & 0x01010101u) * 0x01020408u) >> 24; }
// 4 bits -> 0xFF/0x00 bytes
__device__ __forceinline__ uint32_t unpack4(uint32_t b) { return ((b * 0x00204081u) & 0x01010101u) * 0xFFu; }

template <int CMP>
__device__ __forceinline__ uint32_t pred_bits16(const uint4 &v, uint32_t target) {
    const uint32_t t4 = target * 0x01010101u;
    return pack4(vcmp4<CMP>(v.x, t4)) | (pack4(vcmp4<CMP>(v.y, t4)) << 4) | (pack4(vcmp4<CMP>(v.z, t4)) << 8) |
           (pack4(vcmp4<CMP>(v.w, t4)) << 12);
}
// bits of the lane's 16 bytes [base, base+16) that lie in [lo, hi)
__device__ __forceinline__ uint32_t range_bits(int lo, int hi, int base) {
    int a = lo - base, z = hi - base;
    a = a < 0 ? 0 : a;
    z = z > 16 ? 16 : z;
    if (z <= a) return 0u;
    return ((1u << z) - 1u) & ~((1u << a) - 1u);
}
__device__ __forceinline__ uint4 mask_bytes(const uint4 &v, uint32_t bits16, bool keep_max) {
    // keep bytes whose bit is set; the others become neutral (0 for max, 0xFF for min)
    uint4 m;
    m.x = unpack4(bits16 & 0xF);
    m.y = unpack4((bits16 >> 4) & 0xF);
    m.z = unpack4((bits16 >> 8) & 0xF);
    m.w = unpack4((bits16 >> 12) & 0xF);
    uint4 r;
    if (keep_max) {
        r.x = v.x & m.x; r.y = v.y & m.y; r.z = v.z & m.z; r.w = v.w & m.w;
    } else {
        r.x = v.x | ~m.x; r.y = v.y | ~m.y; r.z = v.z | ~m.z; r.w = v.w | ~m.w;
    }
    return r;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Debug progress words (host-mapped memory set by cdc_debug_progress); null in
// normal runs.  Slot layout: 4 x u64 per warp: {tag|stage, c, s, aux}.
__device__ unsigned long long *g_dbg = nullptr;
__device__ __forceinline__ void dbg_note(uint64_t slot, uint64_t a, uint64_t b, uint64_t c2, uint64_t d) {
    unsigned long long *p = g_dbg;
    if (p != nullptr && lane_id() == 0 && slot < 8192) {
        volatile unsigned long long *q = p + slot * 4;
        q[0] = a; q[1] = b; q[2] = c2; q[3] = d;
    }
}
__device__ __forceinline__ uint64_t dbg_slot() {
    return (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5) + (gridDim.x == 1 ? 4096 : 0);
}

// ---------------------------------------------------------------- warp ring
struct WarpRing {
    uint8_t *buf;   // NST * STAGE bytes, 128-byte aligned
    uint64_t *bar;  // NST mbarriers
};

// Step-local view of one 2 KiB stage held in shared memory.
struct Step {
    const uint8_t *sp;  // stage buffer
    int64_t B;          // stream position of sp[0]
    __device__ __forceinline__ uint4 vec(int blk) const {
        return *reinterpret_cast<const uint4 *>(sp + blk * 512 + lane_id() * 16);
    }
    __device__ __forceinline__ uint32_t byte_at(int64_t pos) const { return sp[pos - B]; }
};

// Extreme (max or min) of the whole stage, per lane (64 bytes per lane).
template <bool MAX>
__device__ __forceinline__ uint32_t step_lane_extreme(const Step &st) {
    uint32_t hi = acc_init<MAX>(), lo = acc_init<MAX>();
#pragma unroll
    for (int b = 0; b < STAGE / 512; ++b) acc16<MAX>(st.vec(b), hi, lo);
    return acc_extreme<MAX>(hi, lo);
}

// Range Scan (§4.2) inside one stage: first position in [lo, hi) whose byte
// satisfies (byte CMP target); returns hi when there is none.
template <int CMP>
__device__ __forceinline__ int64_t step_find(const Step &st, int64_t lo, int64_t hi, uint32_t target) {
    const int rlo = (int)(lo - st.B), rhi = (int)(hi - st.B);
    if (rlo >= rhi) return hi;
    if (rlo == 0 && rhi == STAGE) {
        // fast reject over the whole stage with the extreme tree
        constexpr bool MAX = (CMP == CMP_GT || CMP == CMP_GEQ);
        if constexpr (CMP != CMP_EQ) {
            uint32_t e = step_lane_extreme<MAX>(st);
            bool any;
            if constexpr (CMP == CMP_GT) any = e > target;
            else if constexpr (CMP == CMP_GEQ) any = e >= target;
            else if constexpr (CMP == CMP_LT) any = e < target;
            else any = e <= target;
            if (!__any_sync(0xFFFFFFFFu, any)) return hi;
        }
    }
    const int lane = lane_id();
    for (int b = rlo >> 9; b <= (rhi - 1) >> 9; ++b) {
        uint32_t bits = pred_bits16<CMP>(st.vec(b), target) & range_bits(rlo, rhi, b * 512 + lane * 16);
        uint32_t bal = __ballot_sync(0xFFFFFFFFu, bits != 0);
        if (bal) {
            int L = __ffs(bal) - 1;
            uint32_t mb = __shfl_sync(0xFFFFFFFFu, bits, L);
            return st.B + b * 512 + L * 16 + (__ffs(mb) - 1);
        }
    }
    return hi;
}

// Extreme Byte Search (§4.1) accumulation of [lo, hi) of one stage into the
// lane accumulators (the tree's leaves; the warp reduction is the root).
template <bool MAX>
__device__ __forceinline__ void step_accumulate(const Step &st, int64_t lo, int64_t hi, uint32_t &acc_hi,
                                                uint32_t &acc_lo) {
    const int rlo = (int)(lo - st.B), rhi = (int)(hi - st.B);
    if (rlo >= rhi) return;
    if (rlo == 0 && rhi == STAGE) {
#pragma unroll
        for (int b = 0; b < STAGE / 512; ++b) acc16<MAX>(st.vec(b), acc_hi, acc_lo);
        return;
    }
    const int lane = lane_id();
    for (int b = rlo >> 9; b <= (rhi - 1) >> 9; ++b) {
        uint32_t bits = range_bits(rlo, rhi, b * 512 + lane * 16);
        acc16<MAX>(mask_bytes(st.vec(b), bits, MAX), acc_hi, acc_lo);
    }
}

// ---------------------------------------------------------------- chain engine
//
// run_chain walks the chunk chain of the stream fbase[0..Lf) that begins with
// a chunk at `start` (0 <= start < Lf).  Every boundary e < Lf (the start of
// the next chunk) is passed to emit.boundary(e), which returns true to stop
// the walk; when the chain's last chunk reaches Lf, emit.end() is called.
// Bytes are read only below read_end (the emitter must stop before needing
// more).  All 32 lanes call this with identical arguments.
template <int ALGO, class Emit>
__device__ void run_chain(const WarpRing &R, const uint8_t *__restrict__ fbase, int64_t Lf, int64_t start,
                          int64_t read_end, uint32_t w, uint64_t max_size, uint64_t policy, Emit &emit) {
    const int lane = lane_id();
    if (read_end > Lf) read_end = Lf;
    const uint8_t *g0 = reinterpret_cast<const uint8_t *>(reinterpret_cast<uintptr_t>(fbase + start) &
                                                          ~static_cast<uintptr_t>(15));
    const int64_t B0 = g0 - fbase;
    const int64_t nbytes = ((read_end - B0) + 15) & ~static_cast<int64_t>(15);
    const int64_t nstages = (nbytes + STAGE - 1) / STAGE;

    if (lane == 0) {
        for (int i = 0; i < NST; ++i) mbar_init(&R.bar[i], 1);
        fence_barrier_init();
    }
    __syncwarp();

    int64_t issued = 0;
    auto issue = [&](int64_t k) {
        if (lane == 0) {
            const int slot = (int)(k % NST);
            const int64_t off = k * STAGE;
            const uint32_t bytes = (uint32_t)(nbytes - off < STAGE ? nbytes - off : STAGE);
            mbar_arrive_expect_tx(&R.bar[slot], bytes);
            tma_load_1d(R.buf + slot * STAGE, g0 + off, bytes, &R.bar[slot], policy);
        }
    };
    for (; issued < nstages && issued < NST; ++issued) issue(issued);

    constexpr bool MAX = (ALGO != ALGO_AE_MIN);
    int64_t s = start;                                                           // current chunk start
    int64_t limit = (Lf - s < (int64_t)max_size) ? Lf : s + (int64_t)max_size;  // chunk end bound
    int64_t c = s;                                                               // next byte to examine
    bool stop = false;
    // RAM state
    int phase = 0;  // 0: window [s, s+w); 1: scan for byte >= M
    uint32_t M = 0, acc_hi = acc_init<true>(), acc_lo = acc_init<true>();
    // AE state
    uint32_t ext = 0;
    int64_t t = 0;
    bool pending = true;  // the chunk's first byte is the first target

    if constexpr (ALGO == ALGO_RAM) {
        if (s + (int64_t)w >= Lf) {  // window does not fit: a single final chunk
            emit.end();
            stop = true;
        }
    }

    int64_t k = 0;
    while (!stop && k < nstages) {
        const int slot = (int)(k % NST);
        dbg_note(dbg_slot(), (2ull << 56) | (uint64_t)k, (uint64_t)c, (uint64_t)s, (uint64_t)issued);
        mbar_wait(&R.bar[slot], (uint32_t)((k / NST) & 1));
        Step st{R.buf + slot * STAGE, B0 + k * STAGE};
        const int64_t E = st.B + STAGE;
        dbg_note(dbg_slot(), (1ull << 56) | (uint64_t)k, (uint64_t)c, (uint64_t)s, (uint64_t)nstages);

        while (!stop && c < E) {
            if constexpr (ALGO == ALGO_RAM) {
                if (phase == 0) {
                    const int64_t we = s + (int64_t)w;
                    const int64_t hi = we < E ? we : E;
                    step_accumulate<true>(st, c, hi, acc_hi, acc_lo);
                    c = hi;
                    if (c == we) {
                        M = warp_extreme<true>(acc_extreme<true>(acc_hi, acc_lo));
                        phase = 1;
                    }
                } else {
                    const int64_t hi = limit < E ? limit : E;
                    const int64_t i = step_find<CMP_GEQ>(st, c, hi, M);
                    int64_t e;
                    if (i < hi) e = i + 1;            // boundary byte ends the chunk
                    else if (hi == limit) e = limit;  // cap or end of stream
                    else { c = hi; continue; }
                    if (e >= Lf) { emit.end(); stop = true; break; }
                    if (emit.boundary(e)) { stop = true; break; }
                    s = e; c = e; phase = 0;
                    acc_hi = acc_init<true>(); acc_lo = acc_init<true>();
                    limit = (Lf - s < (int64_t)max_size) ? Lf : s + (int64_t)max_size;
                    if (s + (int64_t)w >= Lf) { emit.end(); stop = true; break; }
                }
            } else {
                if (pending) {  // first byte of the chunk: the first target
                    ext = st.byte_at(c);
                    t = c;
                    ++c;
                    pending = false;
                    continue;
                }
                const int64_t dl = t + (int64_t)w + 1;  // window (t, t+w] ends before dl
                int64_t hi = dl < limit ? dl : limit;
                hi = hi < E ? hi : E;
                int64_t i;
                if (ext == (MAX ? 255u : 0u)) i = hi;  // nothing can beat an absolute extreme
                else i = step_find<MAX ? CMP_GT : CMP_LT>(st, c, hi, ext);
                if (i < hi) {  // a new target inside the window
                    ext = st.byte_at(i);
                    t = i;
                    c = i + 1;
                    continue;
                }
                c = hi;
                int64_t e;
                if (hi == dl && dl <= limit) e = dl;  // target unbeaten over its window
                else if (hi == limit) e = limit;      // cap or end of stream
                else continue;                        // stage exhausted
                if (e >= Lf) { emit.end(); stop = true; break; }
                if (emit.boundary(e)) { stop = true; break; }
                s = e; c = e; pending = true;
                limit = (Lf - s < (int64_t)max_size) ? Lf : s + (int64_t)max_size;
            }
        }
        __syncwarp();
        ++k;
        if (!stop && issued < nstages) {
            issue(issued);
            ++issued;
        }
    }
    // all bytes up to read_end consumed without the emitter stopping: the walk
    // reached the end of the stream (read_end == Lf) inside the last chunk
    if (!stop) {
        if (c >= Lf) emit.end();
        else emit.exhausted(c);
    }
    // drain copies still in flight before the ring is reused or the CTA exits
    dbg_note(dbg_slot(), (3ull << 56) | (uint64_t)k, (uint64_t)c, (uint64_t)s, (uint64_t)issued);
    for (int64_t j = k; j < issued; ++j) mbar_wait(&R.bar[j % NST], (uint32_t)((j / NST) & 1));
    __syncwarp();
    dbg_note(dbg_slot(), (4ull << 56) | (uint64_t)k, (uint64_t)c, (uint64_t)s, (uint64_t)issued);
}

}  // namespace cdc
