// ks_api.cu -- the C ABI of libksort.so (include/ksort.h).  Validates
// arguments the way sort_core does, picks the engine, fills ks_status_t.
#include <cstdio>
#include <cstring>
#include <vector>

#include "ks_host.h"
#include "ks_internal.cuh"

#ifndef KS_GIT
#define KS_GIT "dev"
#endif

using namespace ks;

namespace {

void copy_fast(ks_status_t *s, const FastResult &r)
{
    s->levels = r.levels;
    s->bytes_moved = r.bytes_moved;
    s->keys_partitioned = r.keys_partitioned;
    s->keys_leaf_sorted = r.keys_leaf;
    s->leaves = r.leaves;
    s->launches = r.launches;
    s->host_syncs = r.host_syncs;
    for (int p = 0; p < 8; ++p) {
        s->phase_ms[p] = r.phase_ms[p];
        s->phase_launches[p] = r.phase_launches[p];
        s->phase_bytes[p] = r.phase_bytes[p];
    }
}

void status_init(ks_status_t *s)
{
    if (!s) return;
    std::memset(s, 0, sizeof(*s));
    s->bad_index = -1;
}

// Fetch the offending key for the NonFiniteKeyError message (sort_core.py:58).
void fill_bad(ks_status_t *s, const double *d_keys, long long idx, cudaStream_t st)
{
    s->code = KS_NONFINITE;
    s->bad_index = idx;
    double v = 0.0;
    cudaMemcpyAsync(&v, d_keys + idx, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    s->bad_value = v;
}

size_t exact_bytes(long long n, bool counts) { return exact_layout(n, counts).total; }

int run_exact(double *d_keys, long long n, void *ws, size_t ws_bytes, cudaStream_t st, bool counts,
              ks_status_t *s)
{
    ExactResult r{};
    int rc = exact_sort(d_keys, n, ws, ws_bytes, st, counts, &r);
    if (rc != KS_OK) return rc;
    s->exact_used = 1;
    if (r.bad_index >= 0) {
        fill_bad(s, d_keys, r.bad_index, st);
        return KS_NONFINITE;
    }
    s->levels = r.levels;
    if (counts) {
        s->comparisons = r.comparisons;
        s->moves = r.moves;
        s->max_pending_ranges = r.max_pending;
    }
    return KS_OK;
}

}  // namespace

extern "C" {

const char *ks_version(void) { return "ksort sm_100a " KS_GIT; }

size_t ks_workspace_bytes(int64_t n_total, int64_t n_segments, uint32_t flags)
{
    if (n_total < 0 || n_segments < 0) return 0;
    if (flags & (KS_FLAG_EXACT | KS_FLAG_COUNTS)) {
        size_t a = exact_bytes(n_total, (flags & KS_FLAG_COUNTS) != 0);
        size_t b = heap_workspace_bytes();
        return a > b ? a : b;
    }
    size_t f = fast_layout(n_total, n_segments < 1 ? 1 : n_segments).total;
    return f > 256 ? f : 256;
}

int ks_sort_f64(double *d_keys, int64_t n, void *d_ws, size_t ws_bytes, void *stream, uint32_t flags,
                ks_status_t *h_status)
{
    ks_status_t local;
    ks_status_t *s = h_status ? h_status : &local;
    status_init(s);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n < 0 || (n > 0 && d_keys == nullptr)) return s->code = KS_BAD_ARG;
    if (flags & KS_FLAG_COUNTS) flags |= KS_FLAG_EXACT;
    if (flags & KS_FLAG_EXACT) {
        int rc = run_exact(d_keys, n, d_ws, ws_bytes, st, (flags & KS_FLAG_COUNTS) != 0, s);
        return s->code = rc;
    }
    FastResult r{};
    int rc = fast_sort(d_keys, n, nullptr, 1, d_ws, ws_bytes, st, (flags & KS_FLAG_PROFILE) != 0, &r);
    if (rc != KS_OK) return s->code = rc;
    if (r.bad_index >= 0) {
        fill_bad(s, d_keys, r.bad_index, st);
        return s->code;
    }
    if (r.mixed_zero) {
        // both signed zeros present: only the exact engine reproduces where the
        // reference leaves each of them; the fast pass wrote nothing to d_keys
        if (ws_bytes < exact_bytes(n, false)) return s->code = KS_NEED_EXACT;
        rc = run_exact(d_keys, n, d_ws, ws_bytes, st, false, s);
        return s->code = rc;
    }
    copy_fast(s, r);
    return s->code = KS_OK;
}

int ks_sort_f64_host(double *h_keys, int64_t n, double *d_keys, void *d_ws, size_t ws_bytes, void *stream,
                     uint32_t flags, ks_status_t *h_status)
{
    ks_status_t local;
    ks_status_t *s = h_status ? h_status : &local;
    status_init(s);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n < 0 || (n > 0 && (d_keys == nullptr || h_keys == nullptr))) return s->code = KS_BAD_ARG;
    if (n == 0) return s->code = KS_OK;
    const size_t bytes = 8ull * (size_t)n;
    if (cudaMemcpyAsync(d_keys, h_keys, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return s->code = KS_CUDA_ERROR;
    auto copy_back = [&]() -> int {
        if (cudaMemcpyAsync(h_keys, d_keys, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return KS_CUDA_ERROR;
        return KS_OK;
    };
    if (flags & KS_FLAG_COUNTS) flags |= KS_FLAG_EXACT;
    if (flags & KS_FLAG_EXACT) {
        int rc = run_exact(d_keys, n, d_ws, ws_bytes, st, (flags & KS_FLAG_COUNTS) != 0, s);
        if (rc == KS_OK) rc = copy_back();
        return s->code = rc;
    }
    FastResult r{};
    int rc = fast_sort(d_keys, n, nullptr, 1, d_ws, ws_bytes, st, (flags & KS_FLAG_PROFILE) != 0, &r, h_keys);
    if (rc != KS_OK) return s->code = rc;
    if (r.bad_index >= 0) {
        fill_bad(s, d_keys, r.bad_index, st);
        return s->code;
    }
    if (r.mixed_zero) {
        if (ws_bytes < exact_bytes(n, false)) return s->code = KS_NEED_EXACT;
        rc = run_exact(d_keys, n, d_ws, ws_bytes, st, false, s);
        if (rc == KS_OK) rc = copy_back();
        return s->code = rc;
    }
    copy_fast(s, r);
    return s->code = KS_OK;
}

int ks_sort_f64_segmented(double *d_keys, const int64_t *d_offsets, int64_t n_segments, int64_t n_total,
                          void *d_ws, size_t ws_bytes, void *stream, uint32_t flags, ks_status_t *h_status)
{
    ks_status_t local;
    ks_status_t *s = h_status ? h_status : &local;
    status_init(s);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n_segments < 0 || n_total < 0 || (n_segments > 0 && d_offsets == nullptr)) return s->code = KS_BAD_ARG;
    if (n_segments == 0) return s->code = KS_OK;
    if (flags & KS_FLAG_COUNTS) return s->code = KS_NOT_SUPPORTED;
    bool exact = (flags & KS_FLAG_EXACT) != 0;
    if (!exact) {
        FastResult r{};
        int rc = fast_sort(d_keys, n_total, reinterpret_cast<const long long *>(d_offsets), n_segments, d_ws,
                           ws_bytes, st, (flags & KS_FLAG_PROFILE) != 0, &r);
        if (rc != KS_OK) return s->code = rc;
        if (r.bad_arg) return s->code = KS_BAD_ARG;   // offsets outside [0, n_total] or decreasing
        if (r.bad_index >= 0) {
            fill_bad(s, d_keys, r.bad_index, st);
            return s->code;
        }
        if (!r.mixed_zero) {
            copy_fast(s, r);
            return s->code = KS_OK;
        }
    }
    // exact engine, one segment at a time (rare path: signed zeros or explicit request)
    if (ws_bytes < exact_bytes(n_total, false)) return s->code = exact ? KS_WORKSPACE_SMALL : KS_NEED_EXACT;
    std::vector<long long> off(n_segments + 1);
    if (cudaMemcpyAsync(off.data(), d_offsets, sizeof(long long) * (n_segments + 1), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return s->code = KS_CUDA_ERROR;
    for (int64_t i = 0; i < n_segments; ++i) {
        long long a = off[i], b = off[i + 1];
        if (b < a || a < 0 || b > n_total) return s->code = KS_BAD_ARG;
    }
    // gate all segments before any write (sort_core.py:178 per array)
    if (exact) {
        long long lo = off[0], hi = off[n_segments];
        long long bad = -1;
        if (hi > lo && gate_range(d_keys + lo, hi - lo, d_ws, st, &bad) != KS_OK) return s->code = KS_CUDA_ERROR;
        if (bad >= 0) {
            fill_bad(s, d_keys, lo + bad, st);
            return s->code;
        }
    }
    for (int64_t i = 0; i < n_segments; ++i) {
        long long a = off[i], m = off[i + 1] - off[i];
        if (m < 1) continue;
        ks_status_t tmp;
        status_init(&tmp);
        int rc = run_exact(d_keys + a, m, d_ws, ws_bytes, st, false, &tmp);
        if (rc == KS_NONFINITE) {
            fill_bad(s, d_keys, a + tmp.bad_index, st);
            return s->code;
        }
        if (rc != KS_OK) return s->code = rc;
        if (tmp.levels > s->levels) s->levels = tmp.levels;
    }
    s->exact_used = 1;
    return s->code = KS_OK;
}

int ks_partition_f64(double *d_keys, int64_t n, int64_t left, int64_t right, void *d_ws, size_t ws_bytes,
                     void *stream, int64_t *h_pivot, int32_t *h_flag, ks_status_t *h_status)
{
    ks_status_t local;
    ks_status_t *s = h_status ? h_status : &local;
    status_init(s);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // sort_core.py:157-160
    if (!(0 <= left && left < right && right < n) || d_keys == nullptr) return s->code = KS_BAD_ARG;
    long long out[4] = {0, 0, 0, 0};
    long long bad = -1;
    int rc = exact_partition(d_keys, n, left, right, d_ws, ws_bytes, st, out, &bad);
    if (rc != KS_OK) return s->code = rc;
    s->exact_used = 1;
    if (bad >= 0) {
        fill_bad(s, d_keys, bad, st);
        return s->code;
    }
    if (h_pivot) *h_pivot = out[0];
    if (h_flag) *h_flag = (int32_t)out[1];
    s->comparisons = (uint64_t)out[2];
    s->moves = (uint64_t)out[3];
    return s->code = KS_OK;
}

int ks_heap_sort_f64_exact(double *d_keys, int64_t n, void *d_ws, size_t ws_bytes, void *stream, uint32_t flags,
                           ks_status_t *h_status)
{
    (void)flags;
    ks_status_t local;
    ks_status_t *s = h_status ? h_status : &local;
    status_init(s);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n < 0 || (n > 0 && d_keys == nullptr)) return s->code = KS_BAD_ARG;
    long long bad = -1;
    unsigned long long cmp = 0, mv = 0;
    int rc = heap_sort_exact(d_keys, n, d_ws, ws_bytes, st, &bad, &cmp, &mv);
    if (rc != KS_OK) return s->code = rc;
    s->exact_used = 1;
    if (bad >= 0) {
        fill_bad(s, d_keys, bad, st);
        return s->code;
    }
    s->comparisons = cmp;
    s->moves = mv;
    s->max_pending_ranges = 0;   // heap sort keeps no worklist (sort_core.py:35-36)
    return s->code = KS_OK;
}

int ks_is_sorted_f64(const double *d_keys, int64_t n, void *d_ws, void *stream, int32_t *h_result)
{
    if (n < 0 || !h_result || !d_ws) return KS_BAD_ARG;
    int r = 1;
    int rc = is_sorted_f64(d_keys, n, d_ws, static_cast<cudaStream_t>(stream), &r);
    *h_result = r;
    return rc;
}

int ks_first_nonfinite_f64(const double *d_keys, int64_t n, void *d_ws, void *stream, int64_t *h_index)
{
    if (n < 0 || !h_index || !d_ws || (n > 0 && !d_keys)) return KS_BAD_ARG;
    long long bad = -1;
    const int rc = gate_range(d_keys, n, d_ws, static_cast<cudaStream_t>(stream), &bad);
    *h_index = bad;
    return rc;
}

int ks_generate_f64(double *d_out, int64_t n, uint64_t seed, int32_t kind, void *stream)
{
    if (n < 0 || (n > 0 && !d_out) || (kind != 0 && kind != 1)) return KS_BAD_ARG;
    return generate_f64(d_out, n, seed, kind, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
