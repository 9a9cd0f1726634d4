// ks_host.h -- host-side interfaces between the C ABI (ks_api.cu) and the
// engines (ks_fast.cu, ks_exact.cu, ks_heap.cu, ks_misc.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace ks {

struct FastLayout {
    long long n;
    int seg_cap, lq_cap, sq_cap, small_cap[2], hb_cap, piv_cap, lut_cap, ch_cap, unit_cap;
    long long mat_cap, bsum_cap;
    size_t o_status, o_seg[2], o_lq, o_lq_ready, o_sq, o_sq_ready, o_small[2], o_hb, o_chunk, o_piv, o_lut, o_mat, o_moff, o_bsum, o_units, o_tmp, o_cls, o_check;
    size_t total;
};

struct FastResult {
    int levels;
    long long bad_index;      // -1 if all finite
    int mixed_zero;           // both signed zeros present: rerun in exact mode
    int bad_arg;              // segmented call: invalid offsets (nothing written)
    unsigned long long bytes_moved, keys_partitioned, keys_leaf;
    long long leaves;
    int launches;
    float phase_ms[8];
    int phase_launches[8];
    unsigned long long phase_bytes[8];
    int host_syncs;
};

FastLayout fast_layout(long long n, long long nseg0);
// h_out (optional): host destination of the sorted keys; the copy is queued
// right behind the sort, before the status read (rewritten if more passes run)
int fast_sort(double *keys, long long n, const long long *d_off, long long nseg0, void *ws,
              size_t ws_bytes, cudaStream_t stream, bool profile, FastResult *res, double *h_out = nullptr);

}  // namespace ks

namespace ks {

struct ExactLayout {
    int big_cap, small_cap, log_cap;
    size_t o_status, o_bad, o_big[2], o_small, o_log, o_bl, o_gl, o_out, o_tmp;
    size_t total;
};

struct ExactResult {
    int levels;
    long long bad_index;
    unsigned long long comparisons, moves, max_pending;
};

ExactLayout exact_layout(long long n, bool with_log);
int exact_sort(double *keys, long long n, void *ws, size_t ws_bytes, cudaStream_t stream, bool counts,
               ExactResult *res);
int exact_partition(double *keys, long long n, long long left, long long right, void *ws, size_t ws_bytes,
                    cudaStream_t stream, long long out[4], long long *bad_index);

// ks_heap.cu
int heap_sort_exact(double *keys, long long n, void *ws, size_t ws_bytes, cudaStream_t stream,
                    long long *bad_index, unsigned long long *comparisons, unsigned long long *moves);
size_t heap_workspace_bytes();

// ks_misc.cu
int generate_f64(double *out, long long n, unsigned long long seed, int kind, cudaStream_t stream);
int is_sorted_f64(const double *keys, long long n, void *ws, cudaStream_t stream, int *result);
int gate_range(const double *a, long long n, void *ws, cudaStream_t stream, long long *bad_index);

}  // namespace ks
