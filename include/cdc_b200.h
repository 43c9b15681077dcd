/*
 * cdc_b200.h -- C ABI of the B200 (sm_100a) hashless content-defined chunker.
 *
 * Implements the hot path of PAPER.md (arxiv 2508.05797, "Accelerating Data
 * Chunking in Deduplication Systems using Vector Instructions"): the RAM and
 * AE (AE-Max / AE-Min) boundary rules of §2.1.2, built from the two patterns
 * of §4 -- Extreme Byte Search (§4.1) and Range Scan (§4.2) -- composed as in
 * §4.3.  The output is the list of chunk boundaries (§2.2.2 Eq. 2: chunking
 * throughput = original data size / time to generate all chunk boundaries).
 *
 * Conventions (DESIGN.md §3 lists every reading of the paper):
 *   - A stream is d[0..L).  A chunk starting at s ends at an exclusive offset
 *     e; the next chunk starts at e.  Boundaries are reported as these
 *     exclusive end offsets (uint64, relative to the stream start), in
 *     increasing order; the last one equals L.  An empty stream has none.
 *   - RAM (§2.1.2 l.198): M = max d[s..s+w); the chunk ends after the first
 *     byte at index >= s+w with value >= M.
 *   - AE-Max (§2.1.2 l.169, reading R1): targets are bytes strictly greater
 *     than every earlier byte of the chunk; the chunk ends after the w-byte
 *     window following the first target that no window byte exceeds.
 *     AE-Min mirrors it with "less".
 *   - max_size (reading R5) caps every chunk's length; the minimum chunk size
 *     is the one the window implies (w+1 bytes) -- the paper defines no other.
 *   - Results are bit-identical to the CPU oracle in oracle/ (tests/).
 *
 * Memory: every pointer named d_* is a device pointer (cudaMalloc'ed or a
 * torch CUDA tensor's storage) on the current device; h_* pointers are host
 * memory.  The library never frees caller memory.  Device-side entry points
 * are asynchronous on `stream` (a cudaStream_t passed as void*, NULL = legacy
 * default stream); results are valid after the stream is synchronised.
 * Input buffers may be read up to 15 bytes past their last byte and up to 15
 * bytes before their first byte, never crossing the 16-byte-aligned granule
 * that holds a valid byte (so never a different page).
 *
 * Errors: every function returns 0 on success or a negative cdc_status; the
 * message of the last error on the calling thread is cdc_last_error().
 * Device-side overflow (more boundaries than the caller's capacity) is
 * reported by the count written to d_count exceeding that capacity; the first
 * `capacity` boundaries are still written.
 */
#ifndef CDC_B200_H
#define CDC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDC_ABI_VERSION 1

typedef enum {
    CDC_OK = 0,
    CDC_ERR_INVALID = -1,     /* bad argument (null pointer, w == 0 or >= 2^31, max_size <= w, ...) */
    CDC_ERR_CUDA = -2,        /* a CUDA runtime call failed (message has the CUDA error) */
    CDC_ERR_WORKSPACE = -3,   /* workspace smaller than cdc_workspace_size() */
    CDC_ERR_CAPACITY = -4,    /* host entry point: output capacity too small */
    CDC_ERR_NO_DEVICE = -5    /* no sm_100 device present */
} cdc_status;

/*
 * Algorithms: PAPER.md §2.1.2 (RAM, AE-Max, AE-Min, MAXP).  MAXP (l.173,
 * l.196; §4.3 l.361; readings M1-M5): the chunk from s ends right after the
 * first byte t in [s+h, s+max_size) that is greater than every byte of
 * [t-h, t) and of (t, t+h] (both windows inside the stream), with h = window
 * (at most 65536).  cdc_chunk, cdc_chunk_batch and the host entry points
 * accept it; cdc_chain, cdc_stats, cdc_fetched, cdc_plan_info and
 * cdc_plan_segments (speculative segments) return CDC_ERR_INVALID for it.
 */
typedef enum { CDC_RAM = 0, CDC_AE_MAX = 1, CDC_AE_MIN = 2, CDC_MAXP = 3 } cdc_algo;

/* Extreme Byte Search modes (§4.1) and Range Scan comparators (§4.2). */
typedef enum { CDC_EXT_MAX = 0, CDC_EXT_MIN = 1 } cdc_extreme_mode;
typedef enum { CDC_GT = 0, CDC_GEQ = 1, CDC_LT = 2, CDC_LEQ = 3, CDC_EQ = 4 } cdc_cmp;

typedef struct {
    int32_t  algo;        /* cdc_algo */
    uint32_t window;      /* 1 <= w < 2^31: the fixed-size window of §2.1.2 */
    uint64_t max_size;    /* chunk length cap, > window */
    uint64_t seg_bytes;   /* speculation segment size S (0 = automatic); multiple of 16 */
    uint64_t halo_bytes;  /* max speculative halo walk past a segment end (0 = automatic) */
} cdc_params;

/* Version of this ABI (CDC_ABI_VERSION). */
int cdc_abi_version(void);

/* Message of the last error on the calling thread ("" if none). */
const char *cdc_last_error(void);

/*
 * Window size for a target average chunk size (reading R4):
 * on i.i.d. uniform bytes both RAM and AE chunks average w + 256 bytes when
 * w >> 256 (window, then a geometric wait for the top byte value), so
 * w = avg - 256 for avg >= 512, and w = avg/2 below.  MAXP (reading M5): the
 * smallest h whose local maxima on uniform bytes are at least avg bytes apart
 * on average, 1 / P(h) >= avg with P(h) = sum_v (1/256) (v/256)^(2h)
 * (h = 447 for 8 KiB).  Writes *window.
 */
int cdc_window_for_avg(int32_t algo, uint64_t avg_size, uint32_t *window);

/* Fill *p with defaults for `algo`/`avg_size`: window from
 * cdc_window_for_avg, max_size = 4 * avg_size, automatic S and halo. */
int cdc_params_default(cdc_params *p, int32_t algo, uint64_t avg_size);

/* Upper bound on the number of boundaries of a stream of `len` bytes
 * (every chunk but the last holds >= window+1 bytes). */
uint64_t cdc_max_boundaries(const cdc_params *p, uint64_t len);

/*
 * Workspace (device bytes) needed by cdc_chunk / cdc_chunk_batch for a batch
 * of `nfiles` streams totalling `total_len` bytes whose largest stream has
 * `max_len` bytes (for a single stream pass nfiles = 1 and
 * total_len = max_len = len).  The workspace must be 256-byte aligned and
 * must not be used concurrently by two calls.
 */
int cdc_workspace_size(const cdc_params *p, uint64_t nfiles, uint64_t total_len,
                       uint64_t max_len, size_t *bytes);

/*
 * Chunk one device-resident stream d_data[0..len).
 *   d_bounds : device uint64[bounds_cap]; receives the exclusive chunk end
 *              offsets (ascending, last = len).
 *   d_count  : device uint64[1]; receives the number of boundaries (may
 *              exceed bounds_cap, see overflow above).
 * Asynchronous on `stream`.  The chain is resolved by speculative segments
 * (DESIGN.md §1); when window >= 4096 and the segments are at most 256 KiB,
 * the walkers first try the transfer tables of DESIGN.md §6 (streams whose
 * every chunk step is decided by saturating bytes, e.g. uniform bytes at
 * 8-16 KiB) and fall back to the speculative walk otherwise.  The output is
 * the same either way: PAPER.md §2.1.2's chain, bit for bit.
 */
int cdc_chunk(const cdc_params *p, const uint8_t *d_data, uint64_t len,
              uint64_t *d_bounds, uint64_t bounds_cap, uint64_t *d_count,
              void *d_workspace, size_t workspace_bytes, void *stream);

/*
 * Chunk a packed batch of streams (many-file chunking, BASELINE configs[3]):
 * stream f is d_data[d_file_offsets[f] .. d_file_offsets[f+1]),
 * d_file_offsets is a device uint64[nfiles+1], non-decreasing.
 * Boundaries of stream f are relative to its own start and are written to
 * d_bounds[d_bound_offsets[f] .. d_bound_offsets[f+1]); d_bound_offsets is a
 * device uint64[nfiles+1] written by the call (d_bound_offsets[nfiles] is the
 * total count, also written to d_count).
 */
int cdc_chunk_batch(const cdc_params *p, const uint8_t *d_data,
                    const uint64_t *d_file_offsets, uint64_t nfiles,
                    uint64_t total_len, uint64_t max_len,
                    uint64_t *d_bounds, uint64_t bounds_cap,
                    uint64_t *d_bound_offsets, uint64_t *d_count,
                    void *d_workspace, size_t workspace_bytes, void *stream);

/*
 * End-to-end entry point with HOST buffers: copies h_data to the device,
 * chunks it, copies the boundaries back to h_bounds (host uint64[bounds_cap])
 * and the count to *h_count; synchronous.  Device memory is managed by the
 * library (cached between calls on the calling thread's device).
 * Returns CDC_ERR_CAPACITY (with *h_count set) when bounds_cap is too small.
 */
int cdc_chunk_host(const cdc_params *p, const uint8_t *h_data, uint64_t len,
                   uint64_t *h_bounds, uint64_t bounds_cap, uint64_t *h_count);

/*
 * End-to-end batch entry point with HOST buffers (BASELINE configs[3] end to
 * end): stream f is h_data[h_file_offsets[f] - h_file_offsets[0] ..
 * h_file_offsets[f+1] - h_file_offsets[0]), h_file_offsets a host
 * uint64[nfiles+1], non-decreasing.  The files are cut into up to 8 groups of
 * whole files (about 1 GiB each); group k's host-to-device copy runs on a copy
 * stream while group k-1 is chunked (cdc_chunk_batch per group), then the
 * boundaries come back.  Output as cdc_chunk_batch's, on the host:
 * h_bounds (uint64[bounds_cap]) gets every file's exclusive end offsets
 * relative to its own start, h_bound_offsets (uint64[nfiles+1]) the per-file
 * ranges, *h_count the total.  Synchronous; pinned h_data copies at full PCIe
 * speed.  Device memory is managed by the library (cached per device and
 * calling thread).  Returns CDC_ERR_CAPACITY (with *h_count and
 * h_bound_offsets set) when bounds_cap is too small.
 */
int cdc_chunk_batch_host(const cdc_params *p, const uint8_t *h_data, const uint64_t *h_file_offsets,
                         uint64_t nfiles, uint64_t *h_bounds, uint64_t bounds_cap, uint64_t *h_bound_offsets,
                         uint64_t *h_count);

/*
 * Host-only: the first byte of every speculation segment of a single stream of
 * `len` bytes with these parameters (the plan cdc_chunk uses):
 * writes min(n, starts_cap) starts to starts[] and n to *n_out.
 */
int cdc_plan_segments(const cdc_params *p, uint64_t len, uint64_t *starts, uint64_t starts_cap, uint64_t *n_out);

/*
 * Speculative chain from an arbitrary start (range sharding across GPUs,
 * DESIGN.md §6): treats d_data[0..len) as a stream that may continue past
 * `len` (the caller's shard plus its halo), starts a chunk at `start` and
 * writes every chunk start of that chain, beginning with `start`, up to and
 * including the first start >= stop; when the chain's last chunk ends at
 * len before reaching stop, len is written as the final position.
 *   d_starts : device uint64[starts_cap], d_count : device uint64[1].
 * *d_count receives the number written (capped reading as above); the chain
 * ends at len when the last start plus its chunk reaches len.
 */
int cdc_chain(const cdc_params *p, const uint8_t *d_data, uint64_t len,
              uint64_t start, uint64_t stop, uint64_t *d_starts,
              uint64_t starts_cap, uint64_t *d_count, void *stream);

/*
 * Cross-shard re-synchronisation (range sharding across GPUs):
 * the first element of the ascending device list d_a[0..na) that also occurs
 * in the ascending device list d_b[0..nb).  Writes d_out[0] = its index in
 * d_a (na when there is none) and d_out[1] = its index in d_b (-1 when there
 * is none).  Used with d_a = the chunk starts with which shard r's chain
 * continues past its range, d_b = the starts of shard r+1's own chain: from
 * the first common start on the two chains are identical (content-defined
 * boundaries depend only on the bytes after a chunk start).  na, nb < 2^32.
 * Asynchronous on `stream`.
 */
int cdc_first_common(const int64_t *d_a, uint64_t na, const int64_t *d_b, uint64_t nb, int64_t *d_out,
                     void *stream);

/*
 * Batched Extreme Byte Search (§4.1): for each region r in [0, n),
 * region = d_data[d_off[r] .. d_off[r] + d_len[r]) (d_len[r] >= 1),
 * writes the max (mode CDC_EXT_MAX) or min byte to d_value[r] and its
 * leftmost offset within the region to d_pos[r].  One warp per region.
 */
int cdc_extreme_byte_search(const uint8_t *d_data, const uint64_t *d_off,
                            const uint64_t *d_len, uint64_t n, int32_t mode,
                            uint8_t *d_value, uint64_t *d_pos, void *stream);

/*
 * Batched Range Scan (§4.2): for each region r, writes to d_pos[r] the offset
 * within the region of the first byte b with (b cmp d_target[r]), or
 * d_len[r] if there is none.  Regions may be empty.  One warp per region.
 */
int cdc_range_scan(const uint8_t *d_data, const uint64_t *d_off,
                   const uint64_t *d_len, const uint8_t *d_target, uint64_t n,
                   int32_t cmp, uint64_t *d_pos, void *stream);

/* Number of kernel launches made by the last cdc_chunk / cdc_chunk_batch
 * call on this thread (for bench.py's gpu_launches count). */
int cdc_last_launch_count(void);

/*
 * Per-kernel timing for measurement (bench.py's roofline): while enabled,
 * cdc_chunk / cdc_chunk_batch record CUDA events on their stream around each
 * of their kernels.  cdc_profile_collect synchronises on those events and
 * writes, for the pipeline kernels in order {k_seg_prefix, k_speculate,
 * k_fixup}, the summed milliseconds ms_sum[3] and launch counts launches[3]
 * since the previous collect, and the number of calls; it then forgets them.
 * Host-side bookkeeping per calling thread.  (The interval of a kernel runs
 * from the event before its launch to the event after it.)
 */
int cdc_profile_enable(int on);
int cdc_profile_collect(double *ms_sum, uint64_t *launches, uint64_t *calls);

/* Diagnostics: cdc_profile_query writes, for the 4 events of the last
 * profiled call (before each of the 3 kernels and after the last), 1 if the
 * GPU has reached it, 0 if not (-1: event unused). */
int cdc_profile_query(int *done);

/*
 * Diagnostics of the last call that used workspace d_workspace (same params
 * and sizes as that call): synchronises `stream` and writes to stats[8]:
 *   [0] segments G, [1] segment bytes S, [2] halo cap bytes,
 *   [3] 1 if the fused look-back fast path produced the output, 2 if the
 *       transfer tables did (saturated streams), 0 if k_fixup's resolver and
 *       fix-up walkers ran (with CDC_TDEBUG set in the environment this
 *       call also prints why a transfer-table attempt gave up), 3 if K-phase
 *       speculation did ([0..2] are then its segments, segment bytes and halo
 *       cap, [4..6] its nodes that met another chain / gave up / ended or
 *       were never reached, [7] the chain starts its walkers recorded), 4 if
 *       the dense-index mode did ([0..2] its segments, segment bytes and the
 *       bytes indexed past a segment; [4] = [0], [5..7] = 0), [4] segments
 *       whose chain met the
 *       next segment's chain, [5] segments whose halo walk gave up or was
 *       undecided, [6] segments whose chain skipped a later segment or reached
 *       the stream end from a non-final segment, [7] total halo chunks.
 */
/*
 * Host-only: the speculation geometry a call with these arguments uses:
 * out[0] = segment bytes S, out[1] = halo cap bytes, out[2] = segments of a
 * single stream of max_len bytes (floor(max_len / S), at least 1; segment k
 * starts at k * floor(max_len / n) rounded down to 4 KiB when that quotient is
 * >= 64 KiB, else to 16 B).
 */
int cdc_plan_info(const cdc_params *p, uint64_t nfiles, uint64_t total_len, uint64_t max_len, uint64_t *out);

/*
 * Diagnostics: while d_buf (a device uint64 array of 8 + 7 x segments
 * entries) is set, the kernels record globaltimer stamps.  d_buf[0..7]:
 * k_reset first start / last end, k_speculate first CTA start / first return
 * from its PDL wait / last walker end, k_fixup first CTA start / first return
 * from its PDL wait / last end (the caller presets the "first" slots 0, 2, 3,
 * 5, 6 to ~0 and the "last" slots 1, 4, 7 to 0; a k_fixup that runs the fix-up
 * path leaves slot 7 alone).  Then per segment g, at d_buf[8 + 7g]:
 * {at start, at the end of its body walk (first boundary at or past the
 * segment end; 0 if none), at the end of the walk, at the end of its fused
 * write, SM id | halo chunks << 32, transfer tables: index built, table
 * built}.  A segment the transfer tables resolve reuses the slots as {at
 * start, verdict seen, table published, written, block composed (composers
 * only), index built (scan done for the scanner), table built}.  NULL turns
 * recording off.  Never set during measurements.
 */
int cdc_debug_timing(void *d_buf);

int cdc_stats(const cdc_params *p, uint64_t nfiles, uint64_t total_len, uint64_t max_len,
              const void *d_workspace, uint64_t *stats, void *stream);

/*
 * Bytes that k_speculate's walkers copied from global memory into their
 * shared-memory rings during the last call that used d_workspace (ring
 * stages of the TMA walker plus the sparse walk's regions; DESIGN.md §5's
 * per-unit figure), into *out.  This is what bench.py's roofline divides by
 * the kernel time.  Synchronises `stream`.  Arguments as for cdc_stats.
 * Transfer-table index passes, K-phase walkers and k_fixup's walkers are not
 * counted.
 */
int cdc_fetched(const cdc_params *p, uint64_t nfiles, uint64_t total_len, uint64_t max_len,
                const void *d_workspace, uint64_t *out, void *stream);

/*
 * K-phase speculation: a single stream whose window takes the
 * sparse walk (w >= 4096), with default segments (seg_bytes = halo_bytes = 0;
 * with the dense-index mode off, only when they are too long for the transfer
 * tables) is chunked with k chains per segment, started k-th of a chunk length
 * apart, so that a chain entering a segment meets one of them within a few
 * chunks (the boundaries are the same; only the work differs).  k = -1
 * restores the default (4 chains for windows >= 12 KiB -- AE only below 512 MiB --,
 * else 2, more on streams with fewer segments than walkers; or the CDC_KPHASE
 * environment variable), 0 disables it, 1..8 forces k.  Process-
 * wide; it changes cdc_workspace_size's result, so set it before sizing a
 * workspace.  Returns CDC_ERR_INVALID for other values.
 */
int cdc_set_kphase(int k);

/*
 * Dense-index mode (RAM §2.1.2 l.198 and AE l.169 on streams
 * whose every window holds the saturating byte): a single stream of 1-64 MiB
 * with default segments (seg_bytes = halo_bytes = 0), 4096 <= window <= 24 KiB
 * and max_size >= 2 window + 2 is first tried as one recurrence over the
 * positions of the saturating byte (k_dense_index, k_dense_write); the kernels
 * verify that the stream is saturated everywhere and otherwise hand the call
 * to K-phase speculation and then the ordinary pipeline on the device (the
 * boundaries are the same; only the work differs).  With the mode off, default-
 * segment streams try the transfer tables before K-phase, as before it existed.  on = -1 restores the default (on, or the CDC_DENSE
 * environment variable), 0 disables it, 1 enables it.  Process-wide; it
 * changes cdc_workspace_size's result, so set it before sizing a workspace.
 * Returns CDC_ERR_INVALID for other values.
 */
int cdc_set_dense(int on);

#ifdef __cplusplus
}
#endif

#endif /* CDC_B200_H */
