// MCTransferOperator load matrix R (n_t x n_s) folded on the device (transfer.py:56-110).
//
// From the cached source element of every sample (tt_mc_cache_ids):
//   1. stable segmented sort of each target element's N sample ids;
//   2. one run per (target element, source element): a k x k block
//      W[a][b] = (|T|/N) sum_{samples in run} lam_t,a * lam_s,b, with lam_s recomputed at
//      the sample point, clipped >= 0 and renormalised for ALL samples (transfer.py:84-92);
//   3. stable radix sort of the k*k*runs (row * n_s + col) keys, reduce-by-key;
//   4. CSR row pointers.
// Every step is order-deterministic (stable sorts, fixed reductions): R is bitwise
// reproducible.  apply(field) = R @ coeffs is then one SpMV (tt_spmv_rect).
#include <cub/cub.cuh>
#include "tt_common.cuh"

namespace tt {

struct FoldState {
    int64_t n_rows, n_cols, nnz;
    int64_t* keys;     // unique (row * n_cols + col), sorted
    double* vals;
};

__global__ void iota_mod_kernel(int64_t total, int64_t N, int32_t* __restrict__ out) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < total) out[q] = (int32_t)(q % N);
}

__global__ void seg_offsets_kernel(int64_t E, int64_t N, int64_t* __restrict__ off) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e <= E) off[e] = e * N;
}

__global__ void run_flags_kernel(int64_t total, int64_t N, const int32_t* __restrict__ ids,
                                 int32_t* __restrict__ flags) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= total) return;
    flags[q] = (q % N == 0 || ids[q] != ids[q - 1]) ? 1 : 0;
}

__global__ void run_starts_kernel(int64_t total, const int32_t* __restrict__ flags,
                                  const int32_t* __restrict__ run_id, int64_t* __restrict__ starts) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < total && flags[q]) starts[run_id[q]] = q;
}

template <int D>
__global__ void run_blocks_kernel(int64_t n_runs, int64_t total, int64_t N,
                                  const int64_t* __restrict__ starts, const int32_t* __restrict__ ids,
                                  const int32_t* __restrict__ samp, const double* __restrict__ lam,
                                  const double* __restrict__ t_nodes, const int32_t* __restrict__ t_elems,
                                  const double* __restrict__ t_measure, const double* __restrict__ s_rec,
                                  const int32_t* __restrict__ s_elems, int64_t n_cols,
                                  int64_t* __restrict__ keys, double* __restrict__ vals) {
    constexpr int K = D + 1;
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n_runs) return;
    const int64_t q0 = starts[r];
    const int64_t e = q0 / N;
    int64_t q1 = (r + 1 < n_runs) ? starts[r + 1] : total;
    if (q1 > (e + 1) * N) q1 = (e + 1) * N;
    const int es = ids[q0];
    double v[K][D];
    for (int i = 0; i < K; ++i)
        for (int c = 0; c < D; ++c) v[i][c] = t_nodes[(int64_t)t_elems[e * K + i] * D + c];
    Rec<D> rs;
    load_rec<D>(s_rec, es, rs);
    double W[K][K];
    for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b) W[a][b] = 0.0;
    for (int64_t q = q0; q < q1; ++q) {
        const int64_t j = samp[q];
        double lt[K], x[D], ls[K];
        for (int i = 0; i < K; ++i) lt[i] = lam[j * K + i];
        map_point<D>(lt, v, x);
        bary_from_rec<D>(rs, x, ls);
        double sum = 0.0;
        for (int i = 0; i < K; ++i) ls[i] = ls[i] < 0.0 ? 0.0 : ls[i];
        sum = ls[0] + ls[1];
        for (int i = 2; i < K; ++i) sum += ls[i];
        for (int i = 0; i < K; ++i) ls[i] = ls[i] / sum;
        for (int a = 0; a < K; ++a)
            for (int b = 0; b < K; ++b) W[a][b] = fma(lt[a], ls[b], W[a][b]);
    }
    const double scale = t_measure[e] / (double)N;
    for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b) {
            const int64_t o = r * K * K + a * K + b;
            keys[o] = (int64_t)t_elems[e * K + a] * n_cols + s_elems[(int64_t)es * K + b];
            vals[o] = scale * W[a][b];
        }
}

__global__ void key_to_csr_kernel(int64_t nnz, int64_t n_cols, const int64_t* __restrict__ keys,
                                  unsigned long long* __restrict__ row_counts, int32_t* __restrict__ cols) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    const int64_t row = keys[q] / n_cols;
    cols[q] = (int32_t)(keys[q] - row * n_cols);
    atomicAdd(row_counts + row, 1ull);
}

// y = R x.  LPR lanes per row (R rows hold ~35 entries at C5), rows of a warp contiguous;
// each lane issues its column and value loads 4 at a time before the gathers, so a lane
// keeps ~8 independent loads in flight instead of one dependent chain per entry.
template <int LPR>
__global__ void __launch_bounds__(256) spmv_rect_kernel(int64_t n, const int64_t* __restrict__ rp,
                                                        const int32_t* __restrict__ ci,
                                                        const double* __restrict__ v,
                                                        const double* __restrict__ x, double* __restrict__ y) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t row = t / LPR;
    const int sub = (int)(t % LPR);
    double s = 0.0;
    if (row < n) {
        const int64_t q1 = __ldg(rp + row + 1);
        int64_t q = __ldg(rp + row) + sub;
        for (; q + 3 * LPR < q1; q += 4 * LPR) {
            int c[4];
            double a[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) { c[k] = __ldg(ci + q + k * LPR); a[k] = __ldg(v + q + k * LPR); }
#pragma unroll
            for (int k = 0; k < 4; ++k) s = fma(a[k], __ldg(x + c[k]), s);
        }
        for (; q < q1; q += LPR) s = fma(__ldg(v + q), __ldg(x + __ldg(ci + q)), s);
    }
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (row < n && sub == 0) y[row] = s;
}

template <typename T>
static int dalloc(T** p, size_t n, cudaStream_t s) {
    return cuda_status(cudaMallocAsync((void**)p, sizeof(T) * (n ? n : 1), s), "fold alloc");
}

}  // namespace tt

using namespace tt;

extern "C" int tt_mc_fold(const tt_mesh_t* t, const tt_plan_t* p, const tt_mesh_t* src, const double* src_rec,
                          const int32_t* ids, int64_t* nnz_out, void** handle_out, void* stream) {
    if (!t || !p || !src || !src_rec || !ids || !nnz_out || !handle_out || p->kind != TT_PLAN_SHARED ||
        t->dim != src->dim || p->dim != t->dim || !t->measure) {
        set_error("tt_mc_fold: bad arguments (shared plan, matching dims, target measure required)");
        return TT_ERR_INVALID_PARAMETER;
    }
    auto s = as_stream(stream);
    const int64_t E = t->n_elems, N = p->n_samples, total = E * N;
    const int K = t->dim + 1;
    if (total >= 0x7fffffffLL) {
        set_error("tt_mc_fold: E*N exceeds the int32 sort capacity");
        return TT_ERR_CAPACITY;
    }
    int st = TT_OK;
    int32_t *samp0 = nullptr, *samp1 = nullptr, *ids1 = nullptr, *flags = nullptr, *run_id = nullptr;
    int64_t* offs = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    // 1. per-element stable sort of (id, sample)
    if ((st = dalloc(&samp0, total, s)) || (st = dalloc(&samp1, total, s)) || (st = dalloc(&ids1, total, s)) ||
        (st = dalloc(&offs, E + 1, s)))
        return st;
    iota_mod_kernel<<<grid_for(total, 256), 256, 0, s>>>(total, N, samp0);
    seg_offsets_kernel<<<grid_for(E + 1, 256), 256, 0, s>>>(E, N, offs);
    cub::DeviceSegmentedSort::StableSortPairs(nullptr, tmp_bytes, ids, ids1, samp0, samp1, (int)total, (int)E,
                                              offs, offs + 1, s);
    if ((st = cuda_status(cudaMallocAsync(&tmp, tmp_bytes, s), "fold sort tmp"))) return st;
    cub::DeviceSegmentedSort::StableSortPairs(tmp, tmp_bytes, ids, ids1, samp0, samp1, (int)total, (int)E,
                                              offs, offs + 1, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(samp0, s);
    // 2. runs
    if ((st = dalloc(&flags, total, s)) || (st = dalloc(&run_id, total, s))) return st;
    run_flags_kernel<<<grid_for(total, 256), 256, 0, s>>>(total, N, ids1, flags);
    tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flags, run_id, (int)total, s);
    if ((st = cuda_status(cudaMallocAsync(&tmp, tmp_bytes, s), "fold scan tmp"))) return st;
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags, run_id, (int)total, s);
    cudaFreeAsync(tmp, s);
    int32_t last_id = 0, last_flag = 0;
    cudaMemcpyAsync(&last_id, run_id + total - 1, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&last_flag, flags + total - 1, 4, cudaMemcpyDeviceToHost, s);
    if ((st = cuda_status(cudaStreamSynchronize(s), "fold run count"))) return st;
    const int64_t n_runs = (int64_t)last_id + last_flag;
    int64_t* starts = nullptr;
    if ((st = dalloc(&starts, n_runs, s))) return st;
    run_starts_kernel<<<grid_for(total, 256), 256, 0, s>>>(total, flags, run_id, starts);
    cudaFreeAsync(flags, s);
    cudaFreeAsync(run_id, s);
    // 3. k x k blocks per run -> COO (key, val)
    const int64_t n_coo = n_runs * K * K;
    int64_t *keys0 = nullptr, *keys1 = nullptr;
    double *vals0 = nullptr, *vals1 = nullptr;
    if ((st = dalloc(&keys0, n_coo, s)) || (st = dalloc(&vals0, n_coo, s))) return st;
    if (t->dim == 2)
        run_blocks_kernel<2><<<grid_for(n_runs, 128), 128, 0, s>>>(n_runs, total, N, starts, ids1, samp1, p->lam,
                                                                   t->nodes, t->elems, t->measure, src_rec,
                                                                   src->elems, src->n_nodes, keys0, vals0);
    else
        run_blocks_kernel<3><<<grid_for(n_runs, 128), 128, 0, s>>>(n_runs, total, N, starts, ids1, samp1, p->lam,
                                                                   t->nodes, t->elems, t->measure, src_rec,
                                                                   src->elems, src->n_nodes, keys0, vals0);
    cudaFreeAsync(starts, s);
    cudaFreeAsync(ids1, s);
    cudaFreeAsync(samp1, s);
    cudaFreeAsync(offs, s);
    // 4. stable radix sort by key, reduce by key
    if ((st = dalloc(&keys1, n_coo, s)) || (st = dalloc(&vals1, n_coo, s))) return st;
    int end_bit = 1;
    while (end_bit < 63 && ((int64_t)1 << end_bit) < t->n_nodes * src->n_nodes) ++end_bit;
    tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys0, keys1, vals0, vals1, n_coo, 0, end_bit, s);
    if ((st = cuda_status(cudaMallocAsync(&tmp, tmp_bytes, s), "fold radix tmp"))) return st;
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys0, keys1, vals0, vals1, n_coo, 0, end_bit, s);
    cudaFreeAsync(tmp, s);
    int64_t* n_unique_d = nullptr;
    if ((st = dalloc(&n_unique_d, 1, s))) return st;
    tmp_bytes = 0;
    cub::DeviceReduce::ReduceByKey(nullptr, tmp_bytes, keys1, keys0, vals1, vals0, n_unique_d, cub::Sum(),
                                   n_coo, s);
    if ((st = cuda_status(cudaMallocAsync(&tmp, tmp_bytes, s), "fold reduce tmp"))) return st;
    cub::DeviceReduce::ReduceByKey(tmp, tmp_bytes, keys1, keys0, vals1, vals0, n_unique_d, cub::Sum(), n_coo, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(keys1, s);
    cudaFreeAsync(vals1, s);
    int64_t nnz = 0;
    cudaMemcpyAsync(&nnz, n_unique_d, 8, cudaMemcpyDeviceToHost, s);
    if ((st = cuda_status(cudaStreamSynchronize(s), "fold reduce"))) return st;
    cudaFreeAsync(n_unique_d, s);
    FoldState* h = new FoldState{t->n_nodes, src->n_nodes, nnz, keys0, vals0};
    *nnz_out = nnz;
    *handle_out = h;
    return TT_OK;
}

extern "C" int tt_mc_fold_finish(void* handle, int64_t* row_ptr, int32_t* cols, double* vals, void* stream) {
    if (!handle) {
        set_error("tt_mc_fold_finish: null handle");
        return TT_ERR_INVALID_PARAMETER;
    }
    auto s = as_stream(stream);
    FoldState* h = static_cast<FoldState*>(handle);
    int st = TT_OK;
    unsigned long long* counts = nullptr;
    if ((st = cuda_status(cudaMallocAsync((void**)&counts, sizeof(unsigned long long) * h->n_rows, s), "alloc")))
        return st;
    cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * h->n_rows, s);
    cudaMemsetAsync(row_ptr, 0, sizeof(int64_t), s);
    if (h->nnz)
        key_to_csr_kernel<<<grid_for(h->nnz, 256), 256, 0, s>>>(h->nnz, h->n_cols, h->keys, counts, cols);
    size_t tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, counts, reinterpret_cast<unsigned long long*>(row_ptr + 1),
                                  h->n_rows, s);
    void* tmp = nullptr;
    if ((st = cuda_status(cudaMallocAsync(&tmp, tmp_bytes, s), "alloc"))) return st;
    cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, counts, reinterpret_cast<unsigned long long*>(row_ptr + 1),
                                  h->n_rows, s);
    cudaMemcpyAsync(vals, h->vals, sizeof(double) * h->nnz, cudaMemcpyDeviceToDevice, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(counts, s);
    cudaFreeAsync(h->keys, s);
    cudaFreeAsync(h->vals, s);
    delete h;
    return launch_check("tt_mc_fold_finish");
}

extern "C" int tt_spmv_rect(int64_t n_rows, const int64_t* rp, const int32_t* ci, const double* v,
                            const double* x, double* y, void* stream) {
    if (n_rows == 0) return TT_OK;
    // 8 lanes per row (measured: 16 / 32 lanes 40.5 / 51.9 us at C5, 4 lanes ties 8)
    spmv_rect_kernel<8><<<grid_for(n_rows * 8, 256), 256, 0, as_stream(stream)>>>(n_rows, rp, ci, v, x, y);
    return launch_check("spmv_rect_kernel");
}
