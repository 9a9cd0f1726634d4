/*
 * ksort.h -- C ABI of libksort.so, the B200 (sm_100a) K-sort engine.
 *
 * This is the drop-in boundary for the reference's sort hot path
 * (/root/reference/pkg/src/sortlab/sort_core.py).  Plain pointers and sizes
 * only: device pointers come from the caller's allocator (PyTorch's caching
 * allocator in the Python host layer), the stream is a cudaStream_t passed as
 * void*.  The library never allocates device memory and keeps no global
 * mutable state, so distinct buffers may be sorted concurrently from distinct
 * threads/streams (sort_core contract).
 *
 * Every entry point is synchronous with respect to the host for its status
 * output (it synchronises `stream` once before returning), mirroring the
 * reference's synchronous calls (bench.py:149-151 brackets them with a timer).
 *
 * Return codes (also in ks_status_t.code):
 */
#ifndef KSORT_H
#define KSORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KS_OK 0
#define KS_NONFINITE 1        /* NaN/inf key; user buffer untouched (sort_core.py:50-59,178) */
#define KS_BAD_ARG 2          /* invalid range / sizes (sort_core.py:157-160) */
#define KS_CUDA_ERROR 3
#define KS_WORKSPACE_SMALL 4  /* ws_bytes < ks_workspace_bytes(...) */
#define KS_NOT_SUPPORTED 5
#define KS_NEED_EXACT 6       /* input holds both -0.0 and +0.0: the exact engine is needed and
                                 ws_bytes < ks_workspace_bytes(n, nseg, KS_FLAG_EXACT); keys untouched */

/* flags for ks_sort_f64 / ks_sort_f64_segmented */
#define KS_FLAG_EXACT 1u      /* reproduce the reference's exact K-sort permutation
                                 level by level (needed for op counts and for inputs
                                 holding both -0.0 and +0.0) */
#define KS_FLAG_COUNTS 2u     /* fill ks_status_t.comparisons/moves/max_pending_ranges
                                 (implies KS_FLAG_EXACT) */
#define KS_FLAG_PROFILE 4u    /* time every phase with CUDA events (fast engine) */

typedef struct ks_status {
    int32_t code;               /* KS_* */
    int32_t levels;             /* global partition passes executed */
    int64_t bad_index;          /* first non-finite index when code == KS_NONFINITE */
    double bad_value;           /* its value (NaN/inf) */
    uint64_t comparisons;       /* OpCounts.comparisons (sort_core.py:29-41), COUNTS only */
    uint64_t moves;             /* OpCounts.moves, COUNTS only */
    uint64_t max_pending_ranges;/* OpCounts.max_pending_ranges, COUNTS only */
    uint64_t bytes_moved;       /* algorithmic HBM bytes (reads + writes) of all passes */
    uint64_t keys_partitioned;  /* sum over global passes of keys streamed */
    uint64_t keys_leaf_sorted;  /* keys finished by the on-chip leaf sorter */
    int64_t leaves;             /* leaf segments sorted on chip */
    int32_t exact_used;         /* 1 when the exact (reference-permutation) engine ran */
    int32_t launches;           /* kernels launched by this call */
    /* per-phase telemetry, filled only with KS_FLAG_PROFILE (CUDA events on `stream`):
     * phase 0 gate/init, 1 pivots (segment setup), 2 count, 3 scan, 4 scatter,
     * 5 plan, 6 leaf (on-chip finish + fills), 7 local (one-CTA partition rounds) */
    float phase_ms[8];
    int32_t phase_launches[8];
    uint64_t phase_bytes[8];    /* algorithmic bytes of each phase (reads + writes) */
    int32_t host_syncs;         /* times the call waited for the device (1 = the whole recursion ran
                                 * device-resident behind one status read) */
    int32_t reserved_;
} ks_status_t;

/* Workspace bytes needed to sort n_total keys held in n_segments segments
 * (n_segments = 1 for ks_sort_f64) under `flags`. */
size_t ks_workspace_bytes(int64_t n_total, int64_t n_segments, uint32_t flags);

/* Replaces sort_core.k_sort (sort_core.py:169-217): sort d_keys[0..n) ascending
 * in place.  Rejects NaN/inf before any write (sort_core.py:178). */
int ks_sort_f64(double *d_keys, int64_t n, void *d_ws, size_t ws_bytes, void *stream,
                uint32_t flags, ks_status_t *h_status);

/* Replaces sort_core.k_sort (sort_core.py:169-217) on a HOST array: h_keys[0..n)
 * is copied to the device buffer d_keys (n doubles, caller-allocated), sorted
 * there and copied back into h_keys, all on `stream` with one synchronisation
 * (the copy back is queued behind the sort before the status is read, so the
 * device never waits for the host between the three steps).  Pinned h_keys
 * gives asynchronous copies.  On KS_NONFINITE, KS_NEED_EXACT, KS_BAD_ARG and
 * KS_WORKSPACE_SMALL h_keys keeps its bytes (nothing was written to the device
 * copy); after KS_CUDA_ERROR its contents are undefined.  Same flags, codes and
 * status as ks_sort_f64. */
int ks_sort_f64_host(double *h_keys, int64_t n, double *d_keys, void *d_ws, size_t ws_bytes, void *stream,
                     uint32_t flags, ks_status_t *h_status);

/* Batch entry (new API; the reference bench calls k_sort once per array,
 * bench.py:169-173): sort each segment d_keys[off[s]..off[s+1]) independently,
 * exactly as k_sort would sort it.  d_offsets: device int64[n_segments+1],
 * non-decreasing, off[0] >= 0, off[n_segments] <= n_total; the offsets are
 * validated on the device before any write and violations return KS_BAD_ARG
 * with d_keys untouched. */
int ks_sort_f64_segmented(double *d_keys, const int64_t *d_offsets, int64_t n_segments,
                          int64_t n_total, void *d_ws, size_t ws_bytes, void *stream,
                          uint32_t flags, ks_status_t *h_status);

/* Replaces sort_core.ksort_partition (sort_core.py:146-166): one exact K-sort
 * partition of d_keys[left..right] (inclusive) around key = d_keys[left];
 * same output permutation as sort_core._partition (sort_core.py:81-105).
 * Returns pivot index / flag through h_pivot / h_flag; comparisons and moves of
 * the pass (sort_core.py:108-143) through h_status. */
int ks_partition_f64(double *d_keys, int64_t n, int64_t left, int64_t right, void *d_ws,
                     size_t ws_bytes, void *stream, int64_t *h_pivot, int32_t *h_flag,
                     ks_status_t *h_status);

/* Replaces sort_core.heap_sort (sort_core.py:262-286) in its exact form:
 * the reference's own heap sort run on the device (single sequential lane),
 * with its op counts.  Used when the caller asks for counts or the input holds
 * both signed zeros; otherwise the Python layer routes heap_sort to
 * ks_sort_f64 (identical outputs). */
int ks_heap_sort_f64_exact(double *d_keys, int64_t n, void *d_ws, size_t ws_bytes,
                           void *stream, uint32_t flags, ks_status_t *h_status);

/* Replaces sort_core.is_sorted (sort_core.py:62-67): *h_result = 1 iff
 * non-decreasing.  Needs ks_workspace_bytes(n, 1, 0) bytes of workspace (uses 16). */
int ks_is_sorted_f64(const double *d_keys, int64_t n, void *d_ws, void *stream,
                     int32_t *h_result);

/* Replaces the finiteness checks on ingestion, workload._require_finite
 * (workload.py:129-134) and sort_core._check_finite (sort_core.py:50-59):
 * *h_index = first position holding NaN/+-inf, or -1.  Needs 8 bytes of
 * workspace. */
int ks_first_nonfinite_f64(const double *d_keys, int64_t n, void *d_ws, void *stream, int64_t *h_index);

/* Device twin of workload._bulk_uniform01 (workload.py:68-78):
 * d_out[t] = (mix64(seed + (t+1)*0x9E3779B97F4A7C15) >> 11) * 2^-53.
 * kind 0 = uniform01, kind 1 = dup256 ((u >> 56) / 256, BASELINE configs[4]). */
int ks_generate_f64(double *d_out, int64_t n, uint64_t seed, int32_t kind, void *stream);

/* Library build identity, e.g. "ksort sm_100a <git>". */
const char *ks_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KSORT_H */
