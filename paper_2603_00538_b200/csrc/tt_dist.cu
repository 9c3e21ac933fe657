// Multi-GPU pieces of the coupling step: a row-partitioned Jacobi PCG and the
// row gather / scatter kernels of the partitioned load's exchanges.
//
// Row-partitioned PCG (fem.py:113-152, distributed).  Every rank owns a set of mass-matrix
// rows (the target nodes it owns); its local vector u holds the owned entries followed by
// halo entries (neighbour nodes owned by peers), received every iteration.  The recurrence
// is the Chronopoulos-Gear form of the reference's Jacobi PCG (the same Krylov iterates in
// exact arithmetic) because it needs ONE all-reduce per iteration -- of three scalars:
//
//   update:   p = u + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s;  u = dinv r
//   pack:     send_buf = u[send_idx]                       -> halo exchange (host: NCCL)
//   spmv:     w = A u;  sums = (r.u, w.u, r.r) over own rows   -> all-reduce(sum) (NCCL)
//   scalars:  res = sqrt(r.r)/||b||, best iterate, stop test;  beta = g'/g,
//             alpha = g' / (delta - beta g'/alpha)
//
// The scalars live in device memory (tt_dpcg_state_t): no host round trip per iteration;
// the host checks `done` once per chunk of iterations, and every kernel is a no-op once
// done is set.  Best iterate (fem.py:141-152): the scalars kernel marks an improvement and
// the next update copies x -> best_x before it moves x (tt_dpcg_finish settles the last).
// Local sums are block partials reduced in a fixed order by the last block, and the
// all-reduce runs in a fixed order for a fixed world, so solves are run-to-run
// deterministic.
#include "tt_common.cuh"

namespace tt {

struct DState {
    double alpha, beta, gamma, bnorm, res, best;
    int64_t it, maxiter;
    int32_t done, improved, converged, zero_rhs;
    double tol;
    uint32_t ticket;  // last-block counter of the spmv partial reduction
    int32_t primed;   // the first scalars call (r = b) has run
};
static_assert(sizeof(DState) <= TT_DPCG_STATE_BYTES, "tt_dpcg state size");

constexpr int kDBlock = 256;
constexpr int kDMaxBlocks = 148 * 8;

__global__ void dpcg_start_kernel(tt_dpcg_t a) {
    DState* st = reinterpret_cast<DState*>(a.state);
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) {
        st->alpha = st->beta = st->gamma = st->bnorm = st->res = st->best = 0.0;
        st->it = 0; st->maxiter = a.maxiter; st->tol = a.tol;
        st->done = st->improved = st->converged = st->zero_rhs = 0;
        st->ticket = 0;
        st->primed = 0;
    }
    for (int64_t i = tid; i < a.n_own; i += nt) {
        const double di = 1.0 / a.diag[i];
        const double bi = a.b[i];
        a.dinv[i] = di;
        a.x[i] = 0.0;
        a.best_x[i] = 0.0;
        a.r[i] = bi;
        a.u[i] = di * bi;
        a.p[i] = 0.0;
        a.s[i] = 0.0;
    }
}

__global__ void dpcg_update_kernel(tt_dpcg_t a) {
    const DState* st = reinterpret_cast<const DState*>(a.state);
    if (st->done) return;
    const double alpha = st->alpha, beta = st->beta;
    const bool improved = st->improved != 0;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < a.n_own; i += nt) {
        const double xi = a.x[i];
        if (improved) a.best_x[i] = xi;
        const double pi = a.u[i] + beta * a.p[i];
        const double si = a.w[i] + beta * a.s[i];
        const double ri = a.r[i] - alpha * si;
        a.p[i] = pi;
        a.s[i] = si;
        a.x[i] = xi + alpha * pi;
        a.r[i] = ri;
        a.u[i] = a.dinv[i] * ri;
    }
}

__global__ void dpcg_pack_kernel(tt_dpcg_t a) {
    const DState* st = reinterpret_cast<const DState*>(a.state);
    if (st->done) return;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < a.n_send) a.send_buf[t] = a.u[a.send_idx[t]];
}

// w = A u over the own rows (W/8 lanes per row, each lane 8 ELL entries: two int4 column
// loads and four double2 value loads, then 8 independent gathers of u), and the block
// partials of (r.u, w.u, r.r); the last block to finish sums the partials in block order.
template <int W>
__global__ void __launch_bounds__(kDBlock) dpcg_spmv_kernel(tt_dpcg_t a) {
    DState* st = reinterpret_cast<DState*>(a.state);
    if (st->done) return;
    constexpr int LPR = W / 8;
    __shared__ double sh[3][kDBlock / 32];
    __shared__ bool last;
    constexpr int RPW = 32 / LPR;  // rows per warp and trip (the trip count is warp uniform)
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31, sub = lane % LPR;
    double g = 0.0, d = 0.0, rr = 0.0;
    const double* __restrict__ u = a.u;
    for (int64_t base = warp * RPW; base < a.n_own; base += nwarps * RPW) {
        const int64_t i = base + lane / LPR;
        double wi = 0.0;
        if (i < a.n_own) {
            const int4* cq = reinterpret_cast<const int4*>(a.ell_cols + i * W) + 2 * sub;
            const double2* vq = reinterpret_cast<const double2*>(a.ell_vals + i * W + 8 * sub);
            const int4 c0 = __ldg(cq), c1 = __ldg(cq + 1);
            const double2 a0 = __ldg(vq), a1 = __ldg(vq + 1), a2 = __ldg(vq + 2), a3 = __ldg(vq + 3);
            const double s0 = fma(a1.y, u[c0.w], fma(a1.x, u[c0.z], fma(a0.y, u[c0.y], a0.x * u[c0.x])));
            const double s1 = fma(a3.y, u[c1.w], fma(a3.x, u[c1.z], fma(a2.y, u[c1.y], a2.x * u[c1.x])));
            wi = s0 + s1;
        }
        if constexpr (LPR == 2) wi += __shfl_xor_sync(0xffffffffu, wi, 1);
        if (i < a.n_own && sub == 0) {
            a.w[i] = wi;
            const double ri = a.r[i], ui = u[i];
            g = fma(ri, ui, g);
            d = fma(wi, ui, d);
            rr = fma(ri, ri, rr);
        }
    }
    // block partials (fixed shuffle tree), then the last block reduces them in block order
    for (int off = 16; off > 0; off >>= 1) {
        g += __shfl_xor_sync(0xffffffffu, g, off);
        d += __shfl_xor_sync(0xffffffffu, d, off);
        rr += __shfl_xor_sync(0xffffffffu, rr, off);
    }
    const int w = threadIdx.x >> 5;
    if (lane == 0) { sh[0][w] = g; sh[1][w] = d; sh[2][w] = rr; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[3] = {0.0, 0.0, 0.0};
        for (int k = 0; k < 3; ++k)
            for (int q = 0; q < kDBlock / 32; ++q) t[k] += sh[k][q];
        for (int k = 0; k < 3; ++k) a.part[k * gridDim.x + blockIdx.x] = t[k];
        __threadfence();
        last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    if (threadIdx.x < 3) {
        __threadfence();
        double t = 0.0;
        for (unsigned q = 0; q < gridDim.x; ++q) t += __ldcg(a.part + threadIdx.x * gridDim.x + q);
        a.sums[threadIdx.x] = t;
    }
    if (threadIdx.x == 0) st->ticket = 0;
}

// After the all-reduce of sums: iteration bookkeeping on one thread (fem.py:131-152).
__global__ void dpcg_scalars_kernel(tt_dpcg_t a) {
    DState* st = reinterpret_cast<DState*>(a.state);
    if (st->done) return;
    const double gam = a.sums[0], del = a.sums[1], rr = a.sums[2];
    if (!st->primed) {
        // first call (after start): r = b, u = dinv b, w = A u
        st->primed = 1;
        st->bnorm = sqrt(rr);
        if (st->bnorm == 0.0) {
            st->done = 1; st->converged = 1; st->zero_rhs = 1;
            return;
        }
        st->res = st->best = st->bnorm / st->bnorm;  // ||r0|| / ||b||  (fem.py:136)
        st->gamma = gam;
        st->alpha = gam / del;
        st->beta = 0.0;
        st->improved = 0;
        if (st->maxiter == 0) st->done = 1;
        return;
    }
    st->it += 1;
    const double res = sqrt(rr) / st->bnorm;
    st->res = res;
    st->improved = 0;
    if (res < st->best) {
        st->best = res;
        st->improved = 1;  // x holds the new best: the next update (or finish) copies it
    }
    if (res <= st->tol) {
        st->done = 1;
        st->converged = 1;
        return;
    }
    if (st->it >= st->maxiter) {
        st->done = 1;
        return;
    }
    const double beta = gam / st->gamma;
    st->alpha = gam / (del - beta * gam / st->alpha);
    st->beta = beta;
    st->gamma = gam;
}

__global__ void dpcg_finish_kernel(tt_dpcg_t a, tt_pcg_result_t* res) {
    const DState* st = reinterpret_cast<const DState*>(a.state);
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    if (st->zero_rhs) {
        for (int64_t i = tid; i < a.n_own; i += nt) a.x[i] = 0.0;
    } else if (!st->converged && st->improved) {
        for (int64_t i = tid; i < a.n_own; i += nt) a.best_x[i] = a.x[i];
    }
    if (tid == 0 && res) {
        res->iterations = st->it;
        res->residual = st->res;
        res->best_residual = st->best;
        res->converged = st->converged;
        res->zero_rhs = st->zero_rhs;
    }
}

__global__ void gather_rows_kernel(int64_t n, int k, const int64_t* __restrict__ idx,
                                   const double* __restrict__ src, double* __restrict__ dst) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n * k) return;
    const int64_t t = q / k;
    dst[q] = src[idx[t] * k + (q - t * k)];
}

__global__ void scatter_rows_kernel(int64_t n, int k, const int64_t* __restrict__ idx,
                                    const double* __restrict__ src, double* __restrict__ dst) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n * k) return;
    const int64_t t = q / k;
    dst[idx[t] * k + (q - t * k)] = src[q];
}

static unsigned dgrid(int64_t n) {
    int64_t g = (n + kDBlock - 1) / kDBlock;
    if (g < 1) g = 1;
    if (g > kDMaxBlocks) g = kDMaxBlocks;
    return (unsigned)g;
}

static bool dpcg_ok(const tt_dpcg_t* a) {
    if (!a || a->n_own < 0 || a->n_ext < a->n_own || (a->width != 8 && a->width != 16) || !a->state) {
        set_error("tt_dpcg: bad descriptor (width must be 8 or 16)");
        return false;
    }
    return true;
}

}  // namespace tt

using namespace tt;

extern "C" int64_t tt_dpcg_part_doubles(void) { return 3 * kDMaxBlocks; }

extern "C" int tt_dpcg_start(const tt_dpcg_t* a, void* stream) {
    if (!dpcg_ok(a)) return TT_ERR_INVALID_PARAMETER;
    dpcg_start_kernel<<<dgrid(a->n_own), kDBlock, 0, as_stream(stream)>>>(*a);
    return launch_check("dpcg_start_kernel");
}

extern "C" int tt_dpcg_update(const tt_dpcg_t* a, void* stream) {
    if (!dpcg_ok(a)) return TT_ERR_INVALID_PARAMETER;
    dpcg_update_kernel<<<dgrid(a->n_own), kDBlock, 0, as_stream(stream)>>>(*a);
    return launch_check("dpcg_update_kernel");
}

extern "C" int tt_dpcg_pack(const tt_dpcg_t* a, void* stream) {
    if (!dpcg_ok(a)) return TT_ERR_INVALID_PARAMETER;
    if (a->n_send == 0) return TT_OK;
    dpcg_pack_kernel<<<grid_for(a->n_send, kDBlock), kDBlock, 0, as_stream(stream)>>>(*a);
    return launch_check("dpcg_pack_kernel");
}

extern "C" int tt_dpcg_spmv(const tt_dpcg_t* a, void* stream) {
    if (!dpcg_ok(a)) return TT_ERR_INVALID_PARAMETER;
    const int lpr = a->width / 8;
    const unsigned g = dgrid(a->n_own * lpr);
    if (a->width == 8) dpcg_spmv_kernel<8><<<g, kDBlock, 0, as_stream(stream)>>>(*a);
    else dpcg_spmv_kernel<16><<<g, kDBlock, 0, as_stream(stream)>>>(*a);
    return launch_check("dpcg_spmv_kernel");
}

extern "C" int tt_dpcg_scalars(const tt_dpcg_t* a, void* stream) {
    if (!dpcg_ok(a)) return TT_ERR_INVALID_PARAMETER;
    dpcg_scalars_kernel<<<1, 1, 0, as_stream(stream)>>>(*a);
    return launch_check("dpcg_scalars_kernel");
}

extern "C" int tt_dpcg_finish(const tt_dpcg_t* a, tt_pcg_result_t* result, void* stream) {
    if (!dpcg_ok(a)) return TT_ERR_INVALID_PARAMETER;
    dpcg_finish_kernel<<<dgrid(a->n_own), kDBlock, 0, as_stream(stream)>>>(*a, result);
    return launch_check("dpcg_finish_kernel");
}

extern "C" int tt_gather_rows(int64_t n, int k, const int64_t* idx, const double* src, double* dst,
                              void* stream) {
    if (n < 0 || k < 1) { set_error("tt_gather_rows: bad sizes"); return TT_ERR_INVALID_PARAMETER; }
    if (n == 0) return TT_OK;
    gather_rows_kernel<<<grid_for(n * k, 256), 256, 0, as_stream(stream)>>>(n, k, idx, src, dst);
    return launch_check("gather_rows_kernel");
}

extern "C" int tt_scatter_rows(int64_t n, int k, const int64_t* idx, const double* src, double* dst,
                               void* stream) {
    if (n < 0 || k < 1) { set_error("tt_scatter_rows: bad sizes"); return TT_ERR_INVALID_PARAMETER; }
    if (n == 0) return TT_OK;
    scatter_rows_kernel<<<grid_for(n * k, 256), 256, 0, as_stream(stream)>>>(n, k, idx, src, dst);
    return launch_check("scatter_rows_kernel");
}
