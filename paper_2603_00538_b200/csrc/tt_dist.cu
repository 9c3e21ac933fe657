// Multi-GPU pieces of the coupling step: a row-partitioned Jacobi PCG and the
// row gather / scatter kernels of the partitioned load's exchanges.
//
// Row-partitioned PCG (fem.py:113-152, distributed).  Every rank owns a set of mass-matrix
// rows (the target nodes it owns); its local vector u holds the owned entries followed by
// halo entries (neighbour nodes owned by peers), received every iteration.  The recurrence
// is the Chronopoulos-Gear form of the reference's Jacobi PCG (the same Krylov iterates in
// exact arithmetic) because it needs ONE all-reduce per iteration -- of three scalars.  An
// iteration is two kernels and two collectives:
//
//   update:  scalars from the all-reduced (r.u, w.u, r.r) -- the residual test and best
//            iterate of x, then alpha, beta -- computed redundantly (bitwise alike) by every
//            thread; then for the owned rows p = u + beta p, s = w + beta s, x += alpha p,
//            r -= alpha s, u = dinv r, each new u also written to its send slots
//                                                -> halo all-to-all of the send buffer (NCCL)
//   spmv:    w = A u;  (r.u, w.u, r.r) over the owned rows  -> all-reduce(sum) (NCCL)
//
// The scalar state lives in device memory, ping-ponged between two slots by the update's
// parity (its readers and its one writer never touch the same slot), so the host issues
// iterations without reading anything; it checks `done` once per chunk of iterations (a
// CUDA-graph replay with NCCL), and every kernel is a no-op once done is set.  Best
// iterate (fem.py:141-152): an improved residual copies x -> best_x before x moves.
// Local sums are block partials reduced in a fixed order by the last block, and the
// all-reduce runs in a fixed order for a fixed world, so solves are run-to-run
// deterministic.
#include "tt_common.cuh"

namespace tt {

struct DState {
    double alpha, beta, gamma, bnorm, res, best;
    int64_t it, maxiter;
    int32_t done, converged, zero_rhs, primed;
    double tol;
};
struct DStates {
    DState s[2];       // ping-pong: update with parity q reads s[q], writes s[q ^ 1]
    uint32_t ticket;   // last-block counter of the spmv partial reduction
};
static_assert(sizeof(DStates) <= TT_DPCG_STATE_BYTES, "tt_dpcg state size");

constexpr int kDBlock = 256;
constexpr int kDMaxBlocks = 148 * 8;

__global__ void dpcg_start_kernel(tt_dpcg_t a) {
    DStates* st = reinterpret_cast<DStates*>(a.state);
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) {
        for (int q = 0; q < 2; ++q) {
            DState& s = st->s[q];
            s.alpha = s.beta = s.gamma = s.bnorm = s.res = s.best = 0.0;
            s.it = 0; s.maxiter = a.maxiter; s.tol = a.tol;
            s.done = s.converged = s.zero_rhs = s.primed = 0;
        }
        st->ticket = 0;
    }
    for (int64_t i = tid; i < a.n_own; i += nt) {
        const double di = 1.0 / a.diag[i];
        const double bi = a.b[i];
        const double ui = di * bi;
        a.dinv[i] = di;
        a.x[i] = 0.0;
        a.best_x[i] = 0.0;
        a.r[i] = bi;
        a.u[i] = ui;
        a.p[i] = 0.0;
        a.s[i] = 0.0;
        for (int64_t k = a.send_start[i]; k < a.send_start[i + 1]; ++k) a.send_buf[a.send_pos[k]] = ui;
    }
}

// Iteration bookkeeping from the previous state and the all-reduced sums (fem.py:131-152);
// every thread evaluates it identically.  Returns false when the solve is (now) done.
__device__ __forceinline__ bool dpcg_scalars(const DState& in, const double* sums, DState& out,
                                            bool& improved) {
    out = in;
    improved = false;
    if (in.done) return false;
    const double gam = sums[0], del = sums[1], rr = sums[2];
    if (!in.primed) {
        // first update (after start): r = b, u = dinv b, w = A u
        out.primed = 1;
        out.bnorm = sqrt(rr);
        if (out.bnorm == 0.0) {
            out.done = 1; out.converged = 1; out.zero_rhs = 1;
            return false;
        }
        out.res = out.best = out.bnorm / out.bnorm;  // ||r0|| / ||b||  (fem.py:136)
        out.gamma = gam;
        out.alpha = gam / del;
        out.beta = 0.0;
        if (out.maxiter == 0) { out.done = 1; return false; }
        return true;
    }
    out.it = in.it + 1;
    const double res = sqrt(rr) / in.bnorm;
    out.res = res;
    if (res < in.best) {
        out.best = res;
        improved = true;  // x holds the new best
    }
    if (res <= in.tol) { out.done = 1; out.converged = 1; return false; }
    if (out.it >= in.maxiter) { out.done = 1; return false; }
    const double beta = gam / in.gamma;
    out.alpha = gam / (del - beta * gam / in.alpha);
    out.beta = beta;
    out.gamma = gam;
    return true;
}

__global__ void dpcg_update_kernel(tt_dpcg_t a, int parity) {
    DStates* st = reinterpret_cast<DStates*>(a.state);
    const DState in = st->s[parity];
    DState out;
    bool improved;
    const bool go = dpcg_scalars(in, a.sums, out, improved);
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    // (a finished state propagates: the next update copies it into the other slot)
    if (tid == 0) st->s[parity ^ 1] = out;
    if (!go) {
        // done by this test: settle the best iterate (fem.py:141-152) -- it is x itself when
        // this residual improved; b = 0 returns zeros
        if (!in.done && out.zero_rhs)
            for (int64_t i = tid; i < a.n_own; i += nt) a.x[i] = 0.0;
        else if (!in.done && improved && !out.converged)
            for (int64_t i = tid; i < a.n_own; i += nt) a.best_x[i] = a.x[i];
        return;
    }
    const double alpha = out.alpha, beta = out.beta;
    for (int64_t i = tid; i < a.n_own; i += nt) {
        const double xi = a.x[i];
        if (improved) a.best_x[i] = xi;
        const double pi = a.u[i] + beta * a.p[i];
        const double si = a.w[i] + beta * a.s[i];
        const double ri = a.r[i] - alpha * si;
        const double ui = a.dinv[i] * ri;
        a.p[i] = pi;
        a.s[i] = si;
        a.x[i] = xi + alpha * pi;
        a.r[i] = ri;
        a.u[i] = ui;
        for (int64_t k = a.send_start[i]; k < a.send_start[i + 1]; ++k) a.send_buf[a.send_pos[k]] = ui;
    }
}

// w = A u over the own rows (W/8 lanes per row, each lane 8 ELL entries: two int4 column
// loads and four double2 value loads, then 8 independent gathers of u), and the block
// partials of (r.u, w.u, r.r); the last block to finish sums the partials in block order.
// `parity` = the slot the preceding update wrote.
template <int W>
__global__ void __launch_bounds__(kDBlock) dpcg_spmv_kernel(tt_dpcg_t a, int parity) {
    DStates* st = reinterpret_cast<DStates*>(a.state);
    if (st->s[parity].done) return;
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
    // the last block: every thread sums a fixed strided subset of the block partials, then a
    // fixed shuffle / shared tree (deterministic; a one-thread serial sum of ~1k L2 loads cost
    // 40 us per iteration)
    __threadfence();
    double t[3] = {0.0, 0.0, 0.0};
    for (unsigned q = threadIdx.x; q < gridDim.x; q += kDBlock)
#pragma unroll
        for (int k = 0; k < 3; ++k) t[k] += __ldcg(a.part + k * gridDim.x + q);
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int off = 16; off > 0; off >>= 1) t[k] += __shfl_xor_sync(0xffffffffu, t[k], off);
    __syncthreads();
    if (lane == 0) { sh[0][w] = t[0]; sh[1][w] = t[1]; sh[2][w] = t[2]; }
    __syncthreads();
    if (threadIdx.x < 3) {
        double u2 = 0.0;
        for (int q = 0; q < kDBlock / 32; ++q) u2 += sh[threadIdx.x][q];
        a.sums[threadIdx.x] = u2;
    }
    if (threadIdx.x == 0) st->ticket = 0;
}

__global__ void dpcg_finish_kernel(tt_dpcg_t a, tt_pcg_result_t* res) {
    const DStates* st = reinterpret_cast<const DStates*>(a.state);
    if (blockIdx.x == 0 && threadIdx.x == 0 && res) {
        // once done both slots hold the final state; before, the later one is s[1] or s[0]
        const DState& s = st->s[0].done ? st->s[0] : st->s[1];
        res->iterations = s.it;
        res->residual = s.res;
        res->best_residual = s.best;
        res->converged = s.converged;
        res->zero_rhs = s.zero_rhs;
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
    if (!a || a->n_own < 0 || a->n_ext < a->n_own || (a->width != 8 && a->width != 16) || !a->state ||
        !a->send_start) {
        set_error("tt_dpcg: bad descriptor (width must be 8 or 16, send_start required)");
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

extern "C" int tt_dpcg_update(const tt_dpcg_t* a, int parity, void* stream) {
    if (!dpcg_ok(a) || (parity != 0 && parity != 1)) return TT_ERR_INVALID_PARAMETER;
    dpcg_update_kernel<<<dgrid(a->n_own), kDBlock, 0, as_stream(stream)>>>(*a, parity);
    return launch_check("dpcg_update_kernel");
}

extern "C" int tt_dpcg_spmv(const tt_dpcg_t* a, int parity, void* stream) {
    if (!dpcg_ok(a) || (parity != 0 && parity != 1)) return TT_ERR_INVALID_PARAMETER;
    const int lpr = a->width / 8;
    const unsigned g = dgrid(a->n_own * lpr);
    if (a->width == 8) dpcg_spmv_kernel<8><<<g, kDBlock, 0, as_stream(stream)>>>(*a, parity);
    else dpcg_spmv_kernel<16><<<g, kDBlock, 0, as_stream(stream)>>>(*a, parity);
    return launch_check("dpcg_spmv_kernel");
}

extern "C" int tt_dpcg_finish(const tt_dpcg_t* a, tt_pcg_result_t* result, void* stream) {
    if (!dpcg_ok(a)) return TT_ERR_INVALID_PARAMETER;
    dpcg_finish_kernel<<<1, 32, 0, as_stream(stream)>>>(*a, result);
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

// =====================================================================================
// Peer-memory forms (NVLink / NVSwitch, torch symmetric memory): no NCCL call on the data
// path.  Every rank's exchanged buffers live in one symmetric allocation whose peer
// addresses a kernel reads directly.
// =====================================================================================
#include <cooperative_groups.h>
namespace cgp = cooperative_groups;

namespace tt {

// Owner-side node reduction reading every incidence's contribution from the rank that
// computed it: b[n] = sum over q in [inc_start[n], inc_start[n+1]) of
// ptrs[inc_rank[q]][inc_entry[q]], in that (ascending global (element, vertex)) order --
// the single-GPU np.add.at order, so b is bitwise GPU-count invariant.  Peer values are
// read with ld.global.cv (never a stale L1 line).
__global__ void reduce_nodes_ranked_kernel(int64_t n_nodes, const int64_t* __restrict__ inc_start,
                                           const int32_t* __restrict__ inc_rank,
                                           const int32_t* __restrict__ inc_entry,
                                           const double* const* __restrict__ ptrs, double* __restrict__ b) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= n_nodes) return;
    double s = 0.0;
    for (int64_t q = inc_start[n]; q < inc_start[n + 1]; ++q)
        s = add(s, __ldcv(ptrs[__ldg(inc_rank + q)] + __ldg(inc_entry + q)));
    b[n] = s;
}

// ---- cross-GPU barrier over the symmetric signal pads: pads[q] is rank q's pad (uint32
// slots, one per peer).  Called by every thread of the cooperative grid: the grid syncs,
// thread 0 publishes `epoch` into slot `rank` of every peer's pad (release, system scope) and
// waits until every peer published it into its own pad (acquire), the grid syncs again.  A
// wait longer than ~20 s gives up and raises TT_FLAG_PEER_TIMEOUT (a peer that never arrived)
// instead of hanging the device.
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ bool peer_barrier(cgp::grid_group& grid, uint32_t* const* pads, int rank, int world,
                             uint32_t epoch, int32_t* status) {
    __shared__ int ok;
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        __threadfence_system();
        for (int q = 0; q < world; ++q) st_release_sys(pads[q] + rank, epoch);
        const long long t0 = clock64();
        int good = 1;
        for (int q = 0; q < world && good; ++q)
            while ((int32_t)(ld_acquire_sys(pads[rank] + q) - epoch) < 0) {
                if (clock64() - t0 > 40000000000LL) { good = 0; atomicOr(status, TT_FLAG_PEER_TIMEOUT); break; }
            }
    }
    grid.sync();
    if (threadIdx.x == 0) ok = !(__ldcv(status) & TT_FLAG_PEER_TIMEOUT);
    __syncthreads();
    return ok != 0;
}

struct PeerArgs {
    tt_dpcg_t a;                     // owned rows, ELL with columns < n_own local, >= n_own halo
    const int32_t* __restrict__ halo_owner;   // (n_halo,) rank owning halo column h
    const int32_t* __restrict__ halo_row;     // (n_halo,) that rank's local row
    double* const* __restrict__ sym;          // (world,) symmetric buffers: [u (u_len) | sums 2 x 3]
    uint32_t* const* __restrict__ pads;       // (world,) signal pads
    int64_t u_len;                   // doubles of u per rank in the symmetric buffer
    int rank, world;
    uint32_t* epoch;                 // device: barrier epoch of this rank (persistent)
    int32_t* status;                 // TT_FLAG_PEER_TIMEOUT
    tt_pcg_result_t* res;
};

constexpr int kPBlock = 256;

// block sums of 3 values (valid in thread 0) and the fixed-order grid totals of 3 partial
// arrays part[k * gridDim.x + block] (valid in thread 0 of the calling block)
__device__ __forceinline__ void block_sums3(double (&v)[3], double* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    __syncthreads();
    if (l == 0)
        for (int k = 0; k < 3; ++k) sh[k * 32 + w] = v[k];
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = 0; k < 3; ++k) {
            double t = 0.0;
            for (int q = 0; q < nw; ++q) t += sh[k * 32 + q];
            v[k] = t;
        }
}

__device__ __forceinline__ void grid_totals3(const double* part, double* sh, double (&out)[3]) {
    double t[3] = {0.0, 0.0, 0.0};
    for (unsigned q = threadIdx.x; q < gridDim.x; q += blockDim.x)
        for (int k = 0; k < 3; ++k) t[k] += __ldcg(part + k * gridDim.x + q);
    block_sums3(t, sh);
    for (int k = 0; k < 3; ++k) out[k] = t[k];
}

template <int W>
__global__ void __launch_bounds__(kPBlock, 4) dpcg_peer_kernel(PeerArgs P) {
    cgp::grid_group grid = cgp::this_grid();
    const tt_dpcg_t& a = P.a;
    constexpr int LPR = W / 8;
    constexpr int RPW = 32 / LPR;
    __shared__ double sh[3 * 32];
    __shared__ double tot_s[3];
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, sub = lane % LPR;
    const int64_t warp = tid >> 5, nwarps = nt >> 5;
    double* u = P.sym[P.rank];                       // own u rows (local address)
    double* my_sums = u + P.u_len;                   // [2][3]
    uint32_t epoch = *P.epoch;
    const auto barrier = [&]() { return peer_barrier(grid, P.pads, P.rank, P.world, ++epoch, P.status); };
    // gather of column c of u: own rows locally, halo rows from the owning peer
    const auto ucol = [&](int c) -> double {
        if (c < a.n_own) return u[c];
        const int h = c - (int)a.n_own;
        return __ldcv(P.sym[__ldg(P.halo_owner + h)] + __ldg(P.halo_row + h));
    };
    // w = A u over the owned rows; block partials of (r.u, w.u, r.r) -> this rank's sums slot
    const auto spmv_sums = [&](int parity) {
        double g = 0.0, d = 0.0, rr = 0.0;
        for (int64_t base = warp * RPW; base < a.n_own; base += nwarps * RPW) {
            const int64_t i = base + lane / LPR;
            double wi = 0.0;
            if (i < a.n_own) {
                const int4* cq = reinterpret_cast<const int4*>(a.ell_cols + i * W) + 2 * sub;
                const double2* vq = reinterpret_cast<const double2*>(a.ell_vals + i * W + 8 * sub);
                const int4 c0 = __ldg(cq), c1 = __ldg(cq + 1);
                const double2 a0 = __ldg(vq), a1 = __ldg(vq + 1), a2 = __ldg(vq + 2), a3 = __ldg(vq + 3);
                const double s0 = fma(a1.y, ucol(c0.w), fma(a1.x, ucol(c0.z), fma(a0.y, ucol(c0.y), a0.x * ucol(c0.x))));
                const double s1 = fma(a3.y, ucol(c1.w), fma(a3.x, ucol(c1.z), fma(a2.y, ucol(c1.y), a2.x * ucol(c1.x))));
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
        double v[3] = {g, d, rr};
        block_sums3(v, sh);
        if (threadIdx.x == 0)
            for (int k = 0; k < 3; ++k) a.part[k * gridDim.x + blockIdx.x] = v[k];
        grid.sync();
        if (blockIdx.x == 0) {
            double t[3];
            grid_totals3(a.part, sh, t);
            if (threadIdx.x == 0)
                for (int k = 0; k < 3; ++k) my_sums[parity * 3 + k] = t[k];
        }
    };
    // the world's sums, in rank order (every rank computes the same bits)
    const auto read_totals = [&](int parity, double* t) {
        if (threadIdx.x == 0) {
            double s3[3] = {0.0, 0.0, 0.0};
            for (int q = 0; q < P.world; ++q)
                for (int k = 0; k < 3; ++k) s3[k] += __ldcv(P.sym[q] + P.u_len + parity * 3 + k);
            for (int k = 0; k < 3; ++k) tot_s[k] = s3[k];
        }
        __syncthreads();
        for (int k = 0; k < 3; ++k) t[k] = tot_s[k];
        __syncthreads();
    };
    // ---- init: x = 0, r = b, u = dinv b, p = s = 0
    for (int64_t i = tid; i < a.n_own; i += nt) {
        const double di = 1.0 / a.diag[i];
        const double bi = a.b[i];
        a.dinv[i] = di;
        a.x[i] = 0.0;
        a.best_x[i] = 0.0;
        a.r[i] = bi;
        u[i] = di * bi;
        a.p[i] = 0.0;
        a.s[i] = 0.0;
    }
    bool ok = barrier();                 // every rank's u0 visible
    if (ok) spmv_sums(0);
    ok = ok && barrier();                // every rank's sums visible
    double t[3] = {0.0, 0.0, 0.0};
    if (ok) read_totals(0, t);
    DState st;
    st.alpha = st.beta = st.gamma = st.bnorm = st.res = st.best = 0.0;
    st.it = 0; st.maxiter = a.maxiter; st.tol = a.tol;
    st.done = st.converged = st.zero_rhs = st.primed = 0;
    int parity = 1;
    bool improved = false;
    while (ok) {
        DState nxt;
        const bool go = dpcg_scalars(st, t, nxt, improved);
        st = nxt;
        if (!go) {
            if (st.zero_rhs)
                for (int64_t i = tid; i < a.n_own; i += nt) a.x[i] = 0.0;
            else if (improved && !st.converged)
                for (int64_t i = tid; i < a.n_own; i += nt) a.best_x[i] = a.x[i];
            break;
        }
        const double alpha = st.alpha, beta = st.beta;
        for (int64_t i = tid; i < a.n_own; i += nt) {
            const double xi = a.x[i];
            if (improved) a.best_x[i] = xi;
            const double pi = u[i] + beta * a.p[i];
            const double si = a.w[i] + beta * a.s[i];
            const double ri = a.r[i] - alpha * si;
            a.p[i] = pi;
            a.s[i] = si;
            a.x[i] = xi + alpha * pi;
            a.r[i] = ri;
            u[i] = a.dinv[i] * ri;
        }
        // (the previous barrier ordered every peer's reads of the old u before this write)
        ok = barrier();                  // new u visible
        if (!ok) break;
        spmv_sums(parity);
        ok = barrier();                  // sums visible
        if (!ok) break;
        read_totals(parity, t);
        parity ^= 1;
    }
    if (tid == 0) {
        *P.epoch = epoch;
        if (P.res) {
            P.res->iterations = st.it; P.res->residual = st.res; P.res->best_residual = st.best;
            P.res->converged = ok ? st.converged : 0; P.res->zero_rhs = st.zero_rhs;
        }
    }
}

}  // namespace tt

extern "C" int tt_reduce_nodes_ranked(int64_t n_nodes, const int64_t* inc_start, const int32_t* inc_rank,
                                      const int32_t* inc_entry, const double* const* ptrs, double* b,
                                      void* stream) {
    if (n_nodes < 0 || (n_nodes && (!inc_start || !inc_rank || !inc_entry || !ptrs || !b))) {
        set_error("tt_reduce_nodes_ranked: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (n_nodes == 0) return TT_OK;
    reduce_nodes_ranked_kernel<<<grid_for(n_nodes, 256), 256, 0, as_stream(stream)>>>(
        n_nodes, inc_start, inc_rank, inc_entry, ptrs, b);
    return launch_check("reduce_nodes_ranked_kernel");
}

extern "C" int tt_dpcg_peer_solve(const tt_dpcg_t* a, const int32_t* halo_owner, const int32_t* halo_row,
                                  double* const* sym, uint32_t* const* pads, int64_t u_len, int rank,
                                  int world, uint32_t* epoch, int32_t* status, tt_pcg_result_t* result,
                                  void* stream) {
    if (!a || a->n_own < 0 || (a->width != 8 && a->width != 16) || !sym || !pads || !epoch || !status ||
        rank < 0 || rank >= world || a->n_own > u_len) {
        set_error("tt_dpcg_peer_solve: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    PeerArgs P;
    P.a = *a; P.halo_owner = halo_owner; P.halo_row = halo_row; P.sym = sym; P.pads = pads;
    P.u_len = u_len; P.rank = rank; P.world = world; P.epoch = epoch; P.status = status; P.res = result;
    const void* fn = a->width == 8 ? (const void*)dpcg_peer_kernel<8> : (const void*)dpcg_peer_kernel<16>;
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kPBlock, 0);
    if (per < 1) per = 1;
    int64_t need = (a->n_own * (a->width / 8) + kPBlock - 1) / kPBlock;
    const int64_t maxb = (int64_t)sm_count() * per;
    if (need < 1) need = 1;
    const int blocks = (int)(need < maxb ? need : maxb);
    if ((int64_t)blocks * 3 > tt_dpcg_part_doubles()) { set_error("tt_dpcg_peer_solve: partials"); return TT_ERR_CAPACITY; }
    void* args[] = {&P};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kPBlock), args, 0, as_stream(stream));
    return cuda_status(e, "dpcg_peer_kernel (cooperative launch)");
}
