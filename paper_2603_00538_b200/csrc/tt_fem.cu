// P1 mass matrix (CSR, exactly symmetric) and single-launch Jacobi PCG (fem.py:78-152).
//
// Mass assembly is row-owned: row i is built from node i's incidence list (element
// entries ascending), so every value is a fixed-order sum over ascending elements and
// M[i][j] and M[j][i] are the same sum -- symmetric to the last bit like the reference's
// mirrored upper triangle (fem.py:94-109), with no atomics and no global sort.
//
// PCG runs as ONE cooperative kernel (grid = co-resident blocks on all 148 SMs): the
// CSR and the five vectors of a 1M-element mesh fit in the 126 MB L2, so an iteration
// is three grid-wide barriers around L2-bandwidth vector work instead of ~6 kernel
// launches and a host round-trip for the convergence test.  Dot products are
// per-block partials reduced in a fixed order by every block, so all blocks see the
// identical scalars (uniform control flow) and results are run-to-run deterministic.
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include "tt_common.cuh"

namespace cg = cooperative_groups;

namespace tt {

constexpr int kMaxRow = 256;  // max distinct columns per mass-matrix row

// distinct neighbour nodes of row i (including i), ascending
__device__ int row_columns(int i, int k, const int64_t* __restrict__ inc_start,
                           const int32_t* __restrict__ inc, const int32_t* __restrict__ elems,
                           int* cols) {
    int n = 0;
    for (int64_t q = inc_start[i]; q < inc_start[i + 1]; ++q) {
        const int64_t e = inc[q] / k;
        for (int a = 0; a < k; ++a) {
            const int c = elems[e * k + a];
            // insert into sorted unique list
            int pos = n;
            bool dup = false;
            for (int t = 0; t < n; ++t) {
                if (cols[t] == c) { dup = true; break; }
                if (cols[t] > c) { pos = t; break; }
            }
            if (dup) continue;
            if (n >= kMaxRow) return -1;
            for (int t = n; t > pos; --t) cols[t] = cols[t - 1];
            cols[pos] = c;
            ++n;
        }
    }
    return n;
}

__global__ void mass_count_kernel(int64_t n_nodes, int k, const int64_t* __restrict__ inc_start,
                                  const int32_t* __restrict__ inc, const int32_t* __restrict__ elems,
                                  unsigned long long* __restrict__ lens, int32_t* __restrict__ status) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_nodes) return;
    int cols[kMaxRow];
    int n = row_columns((int)i, k, inc_start, inc, elems, cols);
    if (n < 0) { atomicOr(status, TT_FLAG_CAPACITY); n = 0; }
    lens[i] = (unsigned long long)n;
}

struct LocalMass {
    double m[16];
};

__global__ void mass_fill_kernel(int64_t n_nodes, int k, const int64_t* __restrict__ inc_start,
                                 const int32_t* __restrict__ inc, const int32_t* __restrict__ elems,
                                 const double* __restrict__ measure, LocalMass local,
                                 const int64_t* __restrict__ row_ptr, int32_t* __restrict__ cols_out,
                                 double* __restrict__ vals_out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_nodes) return;
    int cols[kMaxRow];
    int n = row_columns((int)i, k, inc_start, inc, elems, cols);
    if (n < 0) return;
    const int64_t base = row_ptr[i];
    for (int t = 0; t < n; ++t) {
        const int c = cols[t];
        double s = 0.0;
        bool any = false;
        for (int64_t q = inc_start[i]; q < inc_start[i + 1]; ++q) {
            const int64_t ea = inc[q];
            const int64_t e = ea / k;
            const int ai = (int)(ea - e * k);
            int ac = -1;
            for (int a = 0; a < k; ++a)
                if (elems[e * k + a] == c) ac = a;
            if (ac < 0) continue;
            const int lo = ai < ac ? ai : ac, hi = ai < ac ? ac : ai;
            // area * local[lo][hi]: the upper-triangle entry (fem.py:93-100)
            const double v = mul(measure[e], local.m[lo * k + hi]);
            s = any ? add(s, v) : v;
            any = true;
        }
        cols_out[base + t] = c;
        vals_out[base + t] = s;
    }
}

// ------------------------------------------------------------------------- PCG
struct PcgArgs {
    int64_t n;
    const int64_t* __restrict__ rp;
    const int32_t* __restrict__ ci;
    const double* __restrict__ v;
    const double* __restrict__ b;
    double tol;
    int64_t maxiter;
    double* x;
    double* best_x;
    double* r;
    double* z;
    double* p0;     // p double buffer: p_{it} is read from one, p_{it+1} written to the other
    double* p1;
    double* ap;
    double* dinv;
    double* part;   // 3 * gridDim.x partial slots
    tt_pcg_result_t* res;
};

constexpr int kRowG = 4;  // lanes per CSR row in the SpMV (rows have ~7 (2-D) / ~15 (3-D) nnz)

// Row dot product sum_q v[q] * col(ci[q]) for kRowG lanes per row: each lane first
// issues all of its (up to 4) column-index and value loads, then all gathers, so the
// dependent ci -> x[ci] chains of a row overlap (memory-level parallelism).
template <class Col>
__device__ __forceinline__ double row_dot(const int64_t q0, const int64_t q1, const int sub,
                                          const int32_t* __restrict__ ci,
                                          const double* __restrict__ v, Col col) {
    double acc = 0.0;
    int64_t q = q0 + sub;
    for (; q + 3 * kRowG < q1; q += 4 * kRowG) {
        int c[4];
        double a[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) { c[t] = ci[q + t * kRowG]; a[t] = v[q + t * kRowG]; }
        double x[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) x[t] = col(c[t]);
#pragma unroll
        for (int t = 0; t < 4; ++t) acc = fma(a[t], x[t], acc);
    }
    int c[4];
    double a[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const bool ok = q + t * kRowG < q1;
        c[t] = ok ? ci[q + t * kRowG] : -1;
        a[t] = ok ? v[q + t * kRowG] : 0.0;
    }
    double x[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) x[t] = c[t] >= 0 ? col(c[t]) : 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) acc = fma(a[t], x[t], acc);
    return acc;
}

// Block sums of NV values; the totals are valid in warp 0.  sh holds 32 * NV doubles.
template <int NV>
__device__ __forceinline__ void block_sums(double (&v)[NV], double* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k)
        for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    __syncthreads();  // previous readers of sh are done
    if (l == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) sh[k * 32 + w] = v[k];
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double t = l < nw ? sh[k * 32 + l] : 0.0;
            for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
            v[k] = t;
        }
    }
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
    double t[1] = {v};
    block_sums<1>(t, sh);
    return t[0];  // valid in warp 0
}

// Grid totals of NV partial arrays part[k * gridDim.x + block].  Every thread loads one
// partial per array (one L2 round trip instead of gridDim/32 dependent ones), then a
// fixed shuffle/shared-memory tree that every warp of every block evaluates identically,
// so all threads of the grid hold bitwise the same totals with no extra barrier.
template <int NV>
__device__ __forceinline__ void grid_totals(const double* part, double* sh, double (&out)[NV]) {
    const int nb = gridDim.x;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    double t[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) t[k] = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
#pragma unroll
        for (int k = 0; k < NV; ++k) t[k] += __ldcg(part + (int64_t)k * nb + i);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k)
        for (int off = 16; off > 0; off >>= 1) t[k] += __shfl_xor_sync(0xffffffffu, t[k], off);
    __syncthreads();
    if (l == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) sh[k * 32 + w] = t[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double u = l < nw ? sh[k * 32 + l] : 0.0;
        for (int off = 16; off > 0; off >>= 1) u += __shfl_xor_sync(0xffffffffu, u, off);
        out[k] = u;
    }
}

__device__ __forceinline__ double grid_total(const double* part, double* sh) {
    double t[1];
    grid_totals<1>(part, sh, t);
    return t[0];
}

#ifdef TT_PCG_TRACE
// instrumentation build only (-DTT_PCG_TRACE): %globaltimer at the phase boundaries of the
// first 64 iterations, recorded by thread 0 of block 0
__device__ unsigned long long g_pcg_trace[64][6];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PCG_MARK(it, k) if (blockIdx.x == 0 && threadIdx.x == 0 && (it) < 64) g_pcg_trace[it][k] = gtimer()
#else
#define PCG_MARK(it, k) ((void)0)
#endif

// x double-buffering for the best-iterate bookkeeping (fem.py:141-152): the iterate lives
// in X[c], the best iterate in X[bi] (X = {x, best_x}).  An update writes in place unless
// X[c] is the best, then into the other buffer, so no per-iteration copy is needed.  On
// exit the final iterate goes to x and the best to best_x; every thread settles exactly
// the rows it updated (the same tid-strided rows), so no barrier is needed.
__device__ __forceinline__ void settle_iterates(double* x, double* bx, int c, int bi, int64_t n,
                                                int64_t tid, int64_t nthreads) {
    if (c == 0 && bi == 1) return;
    for (int64_t i = tid; i < n; i += nthreads) {
        const double xc = (c == 0 ? x : bx)[i], xb = (bi == 0 ? x : bx)[i];
        x[i] = xc;
        bx[i] = xb;
    }
}

// Jacobi PCG, the reference recurrence (fem.py:131-152), two grid barriers/iteration:
//   A: p_new = z + beta p_old formed on the fly for every gathered column (identical
//      bits in every block), own rows stored; Ap = M p_new; partial p.Ap    | sync
//   B: alpha = rz / p.Ap; x += alpha p; r -= alpha Ap; z = dinv r;
//      partials r.r, r.z                                                   | sync
//   then (every block, no barrier): residual test, best iterate, beta = rz_new / rz.
template <int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) pcg_kernel(PcgArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[3 * 32];
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int nb = gridDim.x;
    double* partA = a.part;
    double* partB = a.part + nb;
    double* partC = a.part + 2 * nb;
    const int64_t n = a.n;

    // init: dinv, x = 0, r = b, z = dinv r, p_old = 0 (so p_1 = z exactly)
    double bb = 0.0, rz_p = 0.0;
    for (int64_t i = tid; i < n; i += nthreads) {
        double d = 0.0;
        for (int64_t q = a.rp[i]; q < a.rp[i + 1]; ++q)
            if (a.ci[q] == i) d = a.v[q];
        const double di = 1.0 / d;
        const double bi = a.b[i];
        a.dinv[i] = di;
        a.x[i] = 0.0;
        a.best_x[i] = 0.0;
        a.r[i] = bi;
        const double zi = di * bi;
        a.z[i] = zi;
        a.p0[i] = 0.0;
        bb += bi * bi;
        rz_p += bi * zi;
    }
    {
        double v[2] = {bb, rz_p};
        block_sums<2>(v, sh);
        if (threadIdx.x == 0) { partB[blockIdx.x] = v[0]; partC[blockIdx.x] = v[1]; }
    }
    grid.sync();
    double tot[2];
    grid_totals<2>(partB, sh, tot);  // partC = partB + gridDim.x
    const double bnorm = sqrt(tot[0]);
    double rz = tot[1];
    if (bnorm == 0.0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.res->iterations = 0; a.res->residual = 0.0; a.res->best_residual = 0.0;
            a.res->converged = 1; a.res->zero_rhs = 1;
        }
        return;
    }
    double best = bnorm / bnorm;  // ||r0|| / ||b||  (fem.py:136)
    double res = best;
    double beta = 0.0;
    constexpr int kRowsPerWarp = 32 / kRowG;
    const int64_t warp_id = tid >> 5, nwarps = nthreads >> 5;
    const int lane = threadIdx.x & 31;
    const int sub = lane % kRowG;
    int xc = 0, xbi = 0;  // current / best iterate buffers (settle_iterates)
    double* p_old = a.p0;
    double* p_new = a.p1;
    for (int64_t it = 0; it < a.maxiter; ++it) {
        // ---- A: p_new = z + beta p_old (on the fly), Ap = M p_new, partial p.Ap
        double pap = 0.0;
        for (int64_t w0 = warp_id * kRowsPerWarp; w0 < n; w0 += nwarps * kRowsPerWarp) {
            const int64_t i = w0 + lane / kRowG;
            double s = 0.0;
            if (i < n) {
                const double* __restrict__ z = a.z;
                const double* __restrict__ po = p_old;
                s = row_dot(a.rp[i], a.rp[i + 1], sub, a.ci, a.v,
                            [&](int c) { return z[c] + beta * po[c]; });
            }
#pragma unroll
            for (int off = kRowG / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (i < n && sub == 0) {
                const double pi = a.z[i] + beta * p_old[i];
                p_new[i] = pi;
                a.ap[i] = s;
                pap += pi * s;
            }
        }
        pap = block_sum(pap, sh);
        if (threadIdx.x == 0) partA[blockIdx.x] = pap;
        grid.sync();
        // ---- B: alpha, x += alpha p, r -= alpha Ap, z = dinv r; partial rr, rz
        const double alpha = rz / grid_total(partA, sh);
        double rr = 0.0, rzn = 0.0;
        const double* xs = xc == 0 ? a.x : a.best_x;  // may alias xw (in-place update)
        const int xw_i = xc == xbi ? 1 - xc : xc;
        double* xw = xw_i == 0 ? a.x : a.best_x;
        for (int64_t i = tid; i < n; i += nthreads) {
            const double pi = p_new[i];
            const double xi = xs[i] + alpha * pi;
            const double ri = a.r[i] - alpha * a.ap[i];
            const double zi = a.dinv[i] * ri;
            xw[i] = xi;
            a.r[i] = ri;
            a.z[i] = zi;
            rr += ri * ri;
            rzn += ri * zi;
        }
        {
            double v[2] = {rr, rzn};
            block_sums<2>(v, sh);
            if (threadIdx.x == 0) { partB[blockIdx.x] = v[0]; partC[blockIdx.x] = v[1]; }
        }
        grid.sync();
        // ---- residual test, best iterate, beta (uniform in every block)
        grid_totals<2>(partB, sh, tot);
        res = sqrt(tot[0]) / bnorm;
        const double rz_new = tot[1];
        xc = xw_i;
        if (res < best) {
            best = res;
            xbi = xc;
        }
        if (res <= a.tol) {
            settle_iterates(a.x, a.best_x, xc, xbi, n, tid, nthreads);
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.res->iterations = it + 1; a.res->residual = res; a.res->best_residual = best;
                a.res->converged = 1; a.res->zero_rhs = 0;
            }
            return;
        }
        beta = rz_new / rz;
        rz = rz_new;
        double* t = p_old; p_old = p_new; p_new = t;
    }
    settle_iterates(a.x, a.best_x, xc, xbi, n, tid, nthreads);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.res->iterations = a.maxiter; a.res->residual = res; a.res->best_residual = best;
        a.res->converged = 0; a.res->zero_rhs = 0;
    }
}

// ---------------------------------------------------------------- ELL variant of the PCG
// Fixed-width rows (width W = 16: every row of these P1 mass matrices has <= 16 entries,
// padding = (row, 0.0)), diagonal stored separately.  4 lanes per row; lane `sub` owns
// entries [4 sub, 4 sub + 4): one int4 column load and two double2 value loads, no row
// pointer round trip, then 4 independent gathers.
__global__ void csr_to_ell_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ v, int W, int32_t* __restrict__ ec,
                                  double* __restrict__ ev, double* __restrict__ diag,
                                  int32_t* __restrict__ status) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t q0 = rp[i], len = rp[i + 1] - q0;
    if (len > W) { atomicOr(status, TT_FLAG_CAPACITY); return; }
    double d = 0.0;
    for (int t = 0; t < W; ++t) {
        const bool in = t < len;
        const int c = in ? ci[q0 + t] : (int)i;
        const double a = in ? v[q0 + t] : 0.0;
        if (in && c == i) d = a;
        if (in && (c - i > 32767 || i - c > 32767)) atomicOr(status, TT_FLAG_WIDE_ROWS);
        ec[i * W + t] = c;
        ev[i * W + t] = a;
    }
    diag[i] = d;
}

struct EllArgs {
    int64_t n;
    const int32_t* __restrict__ ec;
    const double* __restrict__ ev;
    const double* __restrict__ diag;
    const double* __restrict__ b;
    double tol;
    int64_t maxiter;
    double* x;
    double* best_x;
    double* r;
    double* z;
    double* p0;
    double* p1;
    double* ap;
    double* dinv;
    double* part;
    tt_pcg_result_t* res;
    int64_t slab_rows;  // SLAB: rows per block held in shared memory (the rest read from L2)
};

// W/8 lanes per row (W = 16: 2 lanes; W = 8, the 2-D matrices: 1 lane): lane `sub` owns
// entries [8 sub, 8 sub + 8) -> 16 independent gathers in flight per lane and half the
// rows-per-group dependency chain of the 4-lane layout
template <int W, class Col>
__device__ __forceinline__ double ell_row8(const int32_t* __restrict__ ec, const double* __restrict__ ev,
                                           int64_t i, int sub, Col col) {
    const int4* cq = reinterpret_cast<const int4*>(ec + i * W) + 2 * sub;
    const int4 c0 = __ldg(cq), c1 = __ldg(cq + 1);
    const double2* vq = reinterpret_cast<const double2*>(ev + i * W + 8 * sub);
    const double2 a0 = __ldg(vq), a1 = __ldg(vq + 1), a2 = __ldg(vq + 2), a3 = __ldg(vq + 3);
    const double x0 = col(c0.x), x1 = col(c0.y), x2 = col(c0.z), x3 = col(c0.w);
    const double x4 = col(c1.x), x5 = col(c1.y), x6 = col(c1.z), x7 = col(c1.w);
    const double s0 = fma(a1.y, x3, fma(a1.x, x2, fma(a0.y, x1, a0.x * x0)));
    const double s1 = fma(a3.y, x7, fma(a3.x, x6, fma(a2.y, x5, a2.x * x4)));
    return s0 + s1;
}

// SLAB (W/8 lanes per row, contiguous row ranges): the block's rows of the matrix -- all of
// them, or the first a.slab_rows when they do not fit -- stay in shared memory for the whole
// solve instead of being re-read from L2/HBM by every SpMV.  One 80-byte chunk per (row,
// lane): 8 f64 values, then the 8 columns as int16 offsets from the row (|c - i| <= 32767,
// checked by tt_csr_to_ell).  Consecutive lanes read consecutive chunks (stride 5 x 16 B),
// so each quarter-warp LDS.128 touches 8 distinct 16-byte bank groups.
__device__ __forceinline__ double slab_row(const uint4* __restrict__ ch, int64_t i,
                                           const double* __restrict__ z, const double* __restrict__ po,
                                           double beta) {
    const uint4 w0 = ch[0], w1 = ch[1], w2 = ch[2], w3 = ch[3], cw = ch[4];
    const auto dlo = [](uint4 w) { return __hiloint2double((int)w.y, (int)w.x); };
    const auto dhi = [](uint4 w) { return __hiloint2double((int)w.w, (int)w.z); };
    const auto off = [](unsigned u, int h) { return (int)(short)(h ? (u >> 16) : (u & 0xffffu)); };
    int c[8];
    c[0] = (int)i + off(cw.x, 0); c[1] = (int)i + off(cw.x, 1);
    c[2] = (int)i + off(cw.y, 0); c[3] = (int)i + off(cw.y, 1);
    c[4] = (int)i + off(cw.z, 0); c[5] = (int)i + off(cw.z, 1);
    c[6] = (int)i + off(cw.w, 0); c[7] = (int)i + off(cw.w, 1);
    double x[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = z[c[t]] + beta * po[c[t]];
    const double s0 = fma(dhi(w1), x[3], fma(dlo(w1), x[2], fma(dhi(w0), x[1], dlo(w0) * x[0])));
    const double s1 = fma(dhi(w3), x[7], fma(dlo(w3), x[6], fma(dhi(w2), x[5], dlo(w2) * x[4])));
    return s0 + s1;
}

// W/8 lanes per row; every block owns a contiguous row range (neighbour gathers hit its L1).
template <int BLOCK, int MINB, int W, bool SLAB>
__global__ void __launch_bounds__(BLOCK, MINB) pcg_ell_kernel(EllArgs a) {
    constexpr int LPR = W / 8;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[3 * 32];
    extern __shared__ uint4 slab[];  // SLAB: (rows of this block) x 2 chunks x 5 uint4
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int nb = gridDim.x;
    double* partA = a.part;
    double* partB = a.part + nb;
    double* partC = a.part + 2 * nb;
    const int64_t n = a.n;
    if constexpr (SLAB) {
        const int64_t rpb = (n + nb - 1) / nb;
        const int64_t lo = min(n, blockIdx.x * rpb), hi = min(n, lo + min(rpb, a.slab_rows));
        for (int64_t q = threadIdx.x; q < (hi - lo) * LPR; q += BLOCK) {
            const int64_t i = lo + q / LPR;
            const int sub = (int)(q % LPR);
            const int4* cq = reinterpret_cast<const int4*>(a.ec + i * W) + 2 * sub;
            const int4 c0 = __ldg(cq), c1 = __ldg(cq + 1);
            const uint4* vq = reinterpret_cast<const uint4*>(a.ev + i * W + 8 * sub);
            uint4* ch = slab + q * 5;
            ch[0] = __ldg(vq); ch[1] = __ldg(vq + 1); ch[2] = __ldg(vq + 2); ch[3] = __ldg(vq + 3);
            const auto pk = [&](int u, int v) {
                return (unsigned)(unsigned short)(short)(u - (int)i) |
                       ((unsigned)(unsigned short)(short)(v - (int)i) << 16);
            };
            ch[4] = make_uint4(pk(c0.x, c0.y), pk(c0.z, c0.w), pk(c1.x, c1.y), pk(c1.z, c1.w));
        }
        // (the first grid.sync below orders these stores before any SpMV read)
    }
    double bb = 0.0, rz_p = 0.0;
    for (int64_t i = tid; i < n; i += nthreads) {
        const double di = 1.0 / a.diag[i];
        const double bi = a.b[i];
        a.dinv[i] = di;
        a.x[i] = 0.0;
        a.best_x[i] = 0.0;
        a.r[i] = bi;
        const double zi = di * bi;
        a.z[i] = zi;
        a.p0[i] = 0.0;
        bb += bi * bi;
        rz_p += bi * zi;
    }
    {
        double v[2] = {bb, rz_p};
        block_sums<2>(v, sh);
        if (threadIdx.x == 0) { partB[blockIdx.x] = v[0]; partC[blockIdx.x] = v[1]; }
    }
    grid.sync();
    double tot[2];
    grid_totals<2>(partB, sh, tot);  // partC = partB + gridDim.x
    const double bnorm = sqrt(tot[0]);
    double rz = tot[1];
    if (bnorm == 0.0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.res->iterations = 0; a.res->residual = 0.0; a.res->best_residual = 0.0;
            a.res->converged = 1; a.res->zero_rhs = 1;
        }
        return;
    }
    double best = bnorm / bnorm;
    double res = best;
    double beta = 0.0;
    constexpr int RPW = 32 / LPR;  // rows per warp
    const int64_t group = tid / LPR;
    const int sub = threadIdx.x & (LPR - 1);
    int xc = 0, xbi = 0;  // current / best iterate buffers (settle_iterates)
    double* p_old = a.p0;
    double* p_new = a.p1;
    for (int64_t it = 0; it < a.maxiter; ++it) {
        PCG_MARK(it, 0);
        double pap = 0.0;
        // rows are processed by LPR-lane groups; the loop trip count is uniform per warp
        const int64_t rpb = (n + nb - 1) / nb;
        const int64_t r_end = min(n, (blockIdx.x + 1) * rpb);
        const int64_t g_first = blockIdx.x * rpb + (threadIdx.x / LPR & ~(RPW - 1));
        for (int64_t i0 = g_first; i0 < blockIdx.x * rpb + rpb; i0 += BLOCK / LPR) {
            const int64_t i = i0 + (group & (RPW - 1));
            double s = 0.0;
            if (i < r_end) {
                const double* __restrict__ z = a.z;
                const double* __restrict__ po = p_old;
                const auto col = [&](int c) { return z[c] + beta * po[c]; };
                const int64_t li = i - blockIdx.x * rpb;  // row within the block
                if (SLAB && li < a.slab_rows) s = slab_row(slab + (li * LPR + sub) * 5, i, z, po, beta);
                else s = ell_row8<W>(a.ec, a.ev, i, sub, col);
            }
#pragma unroll
            for (int off = 1; off < LPR; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (i < r_end && sub == 0) {
                const double pi = a.z[i] + beta * p_old[i];
                p_new[i] = pi;
                a.ap[i] = s;
                pap += pi * s;
            }
        }
        PCG_MARK(it, 1);
        pap = block_sum(pap, sh);
        if (threadIdx.x == 0) partA[blockIdx.x] = pap;
        grid.sync();
        PCG_MARK(it, 2);
        const double alpha = rz / grid_total(partA, sh);
        PCG_MARK(it, 3);
        double rr = 0.0, rzn = 0.0;
        const double* xs = xc == 0 ? a.x : a.best_x;  // may alias xw (in-place update)
        const int xw_i = xc == xbi ? 1 - xc : xc;
        double* xw = xw_i == 0 ? a.x : a.best_x;
        for (int64_t i = tid; i < n; i += nthreads) {
            const double pi = p_new[i];
            const double xi = xs[i] + alpha * pi;
            const double ri = a.r[i] - alpha * a.ap[i];
            const double zi = a.dinv[i] * ri;
            xw[i] = xi;
            a.r[i] = ri;
            a.z[i] = zi;
            rr += ri * ri;
            rzn += ri * zi;
        }
        PCG_MARK(it, 4);
        {
            double v[2] = {rr, rzn};
            block_sums<2>(v, sh);
            if (threadIdx.x == 0) { partB[blockIdx.x] = v[0]; partC[blockIdx.x] = v[1]; }
        }
        grid.sync();
        PCG_MARK(it, 5);
        grid_totals<2>(partB, sh, tot);
        res = sqrt(tot[0]) / bnorm;
        const double rz_new = tot[1];
        xc = xw_i;
        if (res < best) {
            best = res;
            xbi = xc;
        }
        if (res <= a.tol) {
            settle_iterates(a.x, a.best_x, xc, xbi, n, tid, nthreads);
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.res->iterations = it + 1; a.res->residual = res; a.res->best_residual = best;
                a.res->converged = 1; a.res->zero_rhs = 0;
            }
            return;
        }
        beta = rz_new / rz;
        rz = rz_new;
        double* t = p_old; p_old = p_new; p_new = t;
    }
    settle_iterates(a.x, a.best_x, xc, xbi, n, tid, nthreads);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.res->iterations = a.maxiter; a.res->residual = res; a.res->best_residual = best;
        a.res->converged = 0; a.res->zero_rhs = 0;
    }
}


// ------------------------------------------------------- pipelined PCG (one barrier/iteration)
// Ghysels-Vanroose pipelined Jacobi PCG: the same Krylov iterates as fem.py:131-152 in exact
// arithmetic, with the three inner products of an iteration -- (r,u), (w,u), (r,r) -- reduced
// in ONE grid barrier together with the SpMV that does not depend on them:
//   [barrier: partials of (r_i,u_i), (w_i,u_i), (r_i,r_i)]
//   totals -> residual test / best iterate of x_i;  beta_i = g_i/g_{i-1},
//   alpha_i = g_i / (d_i - beta_i g_i / alpha_{i-1})
//   n = A m_i (m = dinv w, double-buffered: the gathers read m_i while owners write m_{i+1})
//   own rows: z = n + beta z; s = w + beta s; p = u + beta p; x += alpha p; r -= alpha s;
//             w -= alpha z; m_{i+1} = dinv w; partials of the next iteration's three products.
//   u = M^-1 r and q = M^-1 s are formed directly from r and s (Ghysels-Vanroose carry them
//   as recurrences u -= alpha q, q = m + beta q, equal in exact arithmetic): 7 vector loads
//   and 7 stores per row instead of 10 and 9 (C2 solve 0.261 -> 0.234 ms, same iterations)
// The iteration that produces x_{i+1} tests it after the next barrier, so iteration counts,
// the stopping rule (recurrence residual <= tol) and best-iterate tracking are the reference's.
struct PipeArgs {
    int64_t n;
    const int32_t* __restrict__ ec;
    const double* __restrict__ ev;
    const double* __restrict__ diag;
    const double* __restrict__ b;
    double tol;
    int64_t maxiter;
    double* x;
    double* best_x;
    double *r, *u, *w, *z, *q, *s, *p, *m0, *m1, *dinv;
    double* part;
    tt_pcg_result_t* res;
    int64_t slab_rows;
};

__device__ __forceinline__ double slab_row_col(const uint4* __restrict__ ch, int64_t i,
                                               const double* __restrict__ v) {
    const uint4 w0 = ch[0], w1 = ch[1], w2 = ch[2], w3 = ch[3], cw = ch[4];
    const auto dlo = [](uint4 w) { return __hiloint2double((int)w.y, (int)w.x); };
    const auto dhi = [](uint4 w) { return __hiloint2double((int)w.w, (int)w.z); };
    const auto off = [](unsigned u, int h) { return (int)(short)(h ? (u >> 16) : (u & 0xffffu)); };
    const int c0 = (int)i + off(cw.x, 0), c1 = (int)i + off(cw.x, 1);
    const int c2 = (int)i + off(cw.y, 0), c3 = (int)i + off(cw.y, 1);
    const int c4 = (int)i + off(cw.z, 0), c5 = (int)i + off(cw.z, 1);
    const int c6 = (int)i + off(cw.w, 0), c7 = (int)i + off(cw.w, 1);
    const double s0 = fma(dhi(w1), v[c3], fma(dlo(w1), v[c2], fma(dhi(w0), v[c1], dlo(w0) * v[c0])));
    const double s1 = fma(dhi(w3), v[c7], fma(dlo(w3), v[c6], fma(dhi(w2), v[c5], dlo(w2) * v[c4])));
    return s0 + s1;
}

// One lane per row: the lane sums its row's 8-column chunks in order (the recurrence's
// own-row updates then keep every lane busy; 2 lanes per row, where one lane idles through
// the updates: C2 solve 0.222 vs 0.213 ms)
template <int BLOCK, int MINB, int W, bool SLAB>
__global__ void __launch_bounds__(BLOCK, MINB) pcg_pipe_kernel(PipeArgs a) {
    constexpr int CPR = W / 8;     // 8-column chunks per row
    constexpr int LPR = 1;         // lanes per row
    constexpr int CPL = CPR / LPR; // chunks per lane
    constexpr int RPW = 32 / LPR;  // rows per warp
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[3 * 32];
    extern __shared__ uint4 slab[];  // SLAB: (rows of this block) x LPR chunks x 5 uint4
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int nb = gridDim.x;
    // partials (r,u) (w,u) (r,r): two sets of 3 * gridDim.x slots, alternating by iteration
    // (a block that runs ahead must not overwrite partials a slower block is still summing)
    const int64_t n = a.n;
    const int64_t rpb = (n + nb - 1) / nb;
    const int64_t r_lo = blockIdx.x * rpb, r_end = min(n, r_lo + rpb);
    const int64_t group = tid / LPR;
    const int sub = threadIdx.x & (LPR - 1);
    if constexpr (SLAB) {
        const int64_t lo = min(n, r_lo), hi = min(n, lo + min(rpb, a.slab_rows));
        for (int64_t q = threadIdx.x; q < (hi - lo) * CPR; q += BLOCK) {
            const int64_t i = lo + q / CPR;
            const int sb = (int)(q % CPR);
            const int4* cq = reinterpret_cast<const int4*>(a.ec + i * W) + 2 * sb;
            const int4 c0 = __ldg(cq), c1 = __ldg(cq + 1);
            const uint4* vq = reinterpret_cast<const uint4*>(a.ev + i * W + 8 * sb);
            uint4* ch = slab + q * 5;
            ch[0] = __ldg(vq); ch[1] = __ldg(vq + 1); ch[2] = __ldg(vq + 2); ch[3] = __ldg(vq + 3);
            const auto pk = [&](int u, int v) {
                return (unsigned)(unsigned short)(short)(u - (int)i) |
                       ((unsigned)(unsigned short)(short)(v - (int)i) << 16);
            };
            ch[4] = make_uint4(pk(c0.x, c0.y), pk(c0.z, c0.w), pk(c1.x, c1.y), pk(c1.z, c1.w));
        }
    }
    // y_i = sum_j A_ij v_j for the LPR-lane group of row i (all lanes of the warp call it)
    const auto spmv_row = [&](int64_t i, const double* __restrict__ v) -> double {
        double acc = 0.0;
        if (i < r_end) {
            const int64_t li = i - r_lo;
            if (SLAB && li < a.slab_rows) {
                acc = slab_row_col(slab + (li * CPR + sub * CPL) * 5, i, v);
#pragma unroll
                for (int c = 1; c < CPL; ++c) acc += slab_row_col(slab + (li * CPR + sub * CPL + c) * 5, i, v);
            } else {
                acc = ell_row8<W>(a.ec, a.ev, i, sub * CPL, [&](int c) { return v[c]; });
#pragma unroll
                for (int c = 1; c < CPL; ++c) acc += ell_row8<W>(a.ec, a.ev, i, sub * CPL + c, [&](int cc) { return v[cc]; });
            }
        }
#pragma unroll
        for (int off = 1; off < LPR; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        return acc;
    };
    // init: x = 0, r = b, u = dinv b; q = s = p = z = 0
    for (int64_t i = tid; i < n; i += nthreads) {
        const double di = 1.0 / a.diag[i];
        const double bi = a.b[i];
        a.dinv[i] = di;
        a.x[i] = 0.0;
        a.best_x[i] = 0.0;
        a.r[i] = bi;
        a.u[i] = di * bi;
        a.z[i] = 0.0; a.s[i] = 0.0; a.p[i] = 0.0;
    }
    grid.sync();
    // w0 = A u0, m0 = dinv w0, partials of (r0,u0), (w0,u0), (r0,r0)
    {
        double pg = 0.0, pd = 0.0, pr = 0.0;
        for (int64_t i0 = r_lo + (threadIdx.x / LPR & ~(RPW - 1)); i0 < r_lo + rpb; i0 += BLOCK / LPR) {
            const int64_t i = i0 + (group & (RPW - 1));
            const double wi = spmv_row(i, a.u);
            if (i < r_end && sub == 0) {
                const double ri = a.r[i], ui = a.u[i];
                a.w[i] = wi;
                a.m0[i] = a.dinv[i] * wi;
                pg += ri * ui;
                pd += wi * ui;
                pr += ri * ri;
            }
        }
        double v[3] = {pg, pd, pr};
        block_sums<3>(v, sh);
        if (threadIdx.x == 0) { a.part[blockIdx.x] = v[0]; a.part[nb + blockIdx.x] = v[1]; a.part[2 * nb + blockIdx.x] = v[2]; }
    }
    grid.sync();
    double tot[3];
    grid_totals<3>(a.part, sh, tot);
    const double bnorm = sqrt(tot[2]);
    if (bnorm == 0.0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.res->iterations = 0; a.res->residual = 0.0; a.res->best_residual = 0.0;
            a.res->converged = 1; a.res->zero_rhs = 1;
        }
        return;
    }
    double best = bnorm / bnorm;  // ||r0|| / ||b||  (fem.py:136)
    double res = best;
    double gamma_old = 0.0, alpha = 0.0;
    int xc = 0, xbi = 0;  // current / best iterate buffers (settle_iterates)
    for (int64_t it = 0;; ++it) {
        PCG_MARK(it, 0);
        // ---- x_it's residual test (it >= 1), scalars of this iteration
        const double g = tot[0], d = tot[1];
        if (it > 0) {
            res = sqrt(tot[2]) / bnorm;
            if (res < best) {
                best = res;
                xbi = xc;
            }
            if (res <= a.tol) {
                settle_iterates(a.x, a.best_x, xc, xbi, n, tid, nthreads);
                if (blockIdx.x == 0 && threadIdx.x == 0) {
                    a.res->iterations = it; a.res->residual = res; a.res->best_residual = best;
                    a.res->converged = 1; a.res->zero_rhs = 0;
                }
                return;
            }
        }
        if (it == a.maxiter) break;
        const double beta = it > 0 ? g / gamma_old : 0.0;
        alpha = it > 0 ? g / (d - beta * g / alpha) : g / d;
        gamma_old = g;
        const double* __restrict__ m_cur = (it & 1) ? a.m1 : a.m0;
        double* m_nxt = (it & 1) ? a.m0 : a.m1;
        const double* xs = xc == 0 ? a.x : a.best_x;  // may alias xw (in-place update)
        const int xw_i = xc == xbi ? 1 - xc : xc;
        double* xw = xw_i == 0 ? a.x : a.best_x;
        double pg = 0.0, pd = 0.0, pr = 0.0;
        PCG_MARK(it, 1);
#pragma unroll 1
        for (int64_t i0 = r_lo + (threadIdx.x / LPR & ~(RPW - 1)); i0 < r_lo + rpb; i0 += BLOCK / LPR) {
            const int64_t i = i0 + (group & (RPW - 1));
            // u = M^-1 r and q = M^-1 s are formed directly (the recurrences for u and q
            // reproduce them in exact arithmetic): 7 vector loads + 7 stores per row.  The row's
            // own entries are independent of the SpMV: their loads are issued first so their L2
            // latency overlaps the gathers (C2 solve 0.234 -> 0.220 ms)
            const bool own = i < r_end && sub == 0;
            const double di = own ? a.dinv[i] : 0.0, z0 = own ? a.z[i] : 0.0, w0 = own ? a.w[i] : 0.0;
            const double s0 = own ? a.s[i] : 0.0, r0 = own ? a.r[i] : 0.0, p0 = own ? a.p[i] : 0.0;
            const double x0 = own ? xs[i] : 0.0;
            const double ni = spmv_row(i, m_cur);
            if (own) {
                const double zi = ni + beta * z0;
                const double si = w0 + beta * s0;
                const double pi = di * r0 + beta * p0;
                const double xi = x0 + alpha * pi;
                const double ri = r0 - alpha * si;
                const double ui = di * ri;
                const double wi = w0 - alpha * zi;
                a.z[i] = zi; a.s[i] = si; a.p[i] = pi;
                xw[i] = xi; a.r[i] = ri; a.w[i] = wi;
                m_nxt[i] = di * wi;
                pg += ri * ui;
                pd += wi * ui;
                pr += ri * ri;
            }
        }
        xc = xw_i;
        PCG_MARK(it, 2);
        double* partG = a.part + ((it + 1) & 1) * 3 * nb;
        double v[3] = {pg, pd, pr};
        block_sums<3>(v, sh);
        if (threadIdx.x == 0) { partG[blockIdx.x] = v[0]; partG[nb + blockIdx.x] = v[1]; partG[2 * nb + blockIdx.x] = v[2]; }
        PCG_MARK(it, 3);
        grid.sync();
        PCG_MARK(it, 4);
        grid_totals<3>(partG, sh, tot);
        PCG_MARK(it, 5);
    }
    settle_iterates(a.x, a.best_x, xc, xbi, n, tid, nthreads);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.res->iterations = a.maxiter; a.res->residual = res; a.res->best_residual = best;
        a.res->converged = 0; a.res->zero_rhs = 0;
    }
}

__global__ void spmv_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, const double* __restrict__ x,
                            double* __restrict__ y) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t i = tid / kRowG;
    const int sub = threadIdx.x % kRowG;
    double s = 0.0;
    if (i < n)
        for (int64_t q = rp[i] + sub; q < rp[i + 1]; q += kRowG) s += v[q] * __ldg(x + ci[q]);
#pragma unroll
    for (int off = kRowG / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (i < n && sub == 0) y[i] = s;
}

// integral of a P1 field: sum_e |T| * (c . w), w = rule.points^T rule.weights (fem.py:155-161)
__global__ void integrate_kernel(int64_t E, int k, const int32_t* __restrict__ elems,
                                 const double* __restrict__ measure, const double* __restrict__ c,
                                 LocalMass w, double* __restrict__ part) {
    __shared__ double sh[33];
    double s = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        double t = 0.0;
        for (int a = 0; a < k; ++a) t += c[elems[e * k + a]] * w.m[a];
        s += measure[e] * t;
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_parts_kernel(int nparts, const double* __restrict__ part, double* __restrict__ out) {
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (int i = threadIdx.x; i < nparts; i += 32) t += part[i];
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (threadIdx.x == 0) *out = t;
    }
}

template <int BLOCK, int MINB>
static int pcg_launch(PcgArgs& a, int64_t n, cudaStream_t st) {
    static const int per_sm = [] {
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, pcg_kernel<BLOCK, MINB>, BLOCK, 0);
        return per < 1 ? 1 : per;
    }();
    int64_t maxb = (int64_t)sm_count() * per_sm;
    int64_t need = (n * kRowG + BLOCK - 1) / BLOCK;
    if (need < 1) need = 1;
    int blocks = (int)(need < maxb ? need : maxb);
    if (blocks > 148 * 32) blocks = 148 * 32;
    void* args[] = {&a};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)pcg_kernel<BLOCK, MINB>, dim3(blocks), dim3(BLOCK),
                                                args, 0, st);
    return cuda_status(e, "pcg_kernel (cooperative launch)");
}

}  // namespace tt

using namespace tt;

extern "C" int tt_mass_pattern(const tt_mesh_t* m, const int64_t* inc_start, const int32_t* inc,
                               int64_t* row_ptr, int32_t* status, void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3)) {
        set_error("tt_mass_pattern: bad mesh");
        return TT_ERR_INVALID_PARAMETER;
    }
    auto s = as_stream(stream);
    const int k = m->dim + 1;
    unsigned long long* lens = nullptr;
    int st = cuda_status(cudaMallocAsync((void**)&lens, sizeof(unsigned long long) * (m->n_nodes + 1), s),
                         "mass lens alloc");
    if (st) return st;
    cudaMemsetAsync(row_ptr, 0, sizeof(int64_t), s);
    if (m->n_nodes)
        mass_count_kernel<<<grid_for(m->n_nodes, 128), 128, 0, s>>>(m->n_nodes, k, inc_start, inc,
                                                                    m->elems, lens, status);
    size_t tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, lens,
                                  reinterpret_cast<unsigned long long*>(row_ptr + 1), m->n_nodes, s);
    void* tmp = nullptr;
    st = cuda_status(cudaMallocAsync(&tmp, tmp_bytes, s), "scan tmp alloc");
    if (!st) {
        cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, lens,
                                      reinterpret_cast<unsigned long long*>(row_ptr + 1), m->n_nodes, s);
        st = launch_check("mass pattern");
        cudaFreeAsync(tmp, s);
    }
    cudaFreeAsync(lens, s);
    return st;
}

extern "C" int tt_mass_fill(const tt_mesh_t* m, const int64_t* inc_start, const int32_t* inc,
                            const double* local_host, const int64_t* row_ptr, int32_t* cols,
                            double* vals, void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3) || !m->measure || !local_host) {
        set_error("tt_mass_fill: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    const int k = m->dim + 1;
    LocalMass lm;
    for (int i = 0; i < 16; ++i) lm.m[i] = i < k * k ? local_host[i] : 0.0;
    if (m->n_nodes)
        mass_fill_kernel<<<grid_for(m->n_nodes, 128), 128, 0, as_stream(stream)>>>(
            m->n_nodes, k, inc_start, inc, m->elems, m->measure, lm, row_ptr, cols, vals);
    return launch_check("mass_fill_kernel");
}

extern "C" int64_t tt_pcg_workspace_doubles(int64_t n) { return 10 * n + 6 * 148 * 32 + 64; }

extern "C" int tt_pcg(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                      const double* b, double tol, int64_t maxiter, double* x, double* best_x,
                      double* work, tt_pcg_result_t* result, void* stream) {
    if (n < 1 || maxiter < 0) {
        set_error("tt_pcg: bad size");
        return TT_ERR_INVALID_PARAMETER;
    }
    PcgArgs a;
    a.n = n; a.rp = rp; a.ci = ci; a.v = v; a.b = b; a.tol = tol; a.maxiter = maxiter;
    a.x = x; a.best_x = best_x;
    a.r = work; a.z = work + n; a.p0 = work + 2 * n; a.p1 = work + 3 * n; a.ap = work + 4 * n;
    a.dinv = work + 5 * n;
    a.part = work + 6 * n;
    a.res = result;
    // block shape: 2 x 512 threads per SM (measured best of 256x4 / 512x2 / 1024x1)
    return pcg_launch<512, 2>(a, n, as_stream(stream));
}

extern "C" int tt_spmv(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                       const double* x, double* y, void* stream) {
    if (n == 0) return TT_OK;
    spmv_kernel<<<grid_for(n * kRowG, 256), 256, 0, as_stream(stream)>>>(n, rp, ci, v, x, y);
    return launch_check("spmv_kernel");
}

extern "C" int tt_integrate_p1(const tt_mesh_t* m, const double* coeffs, double* out, void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3) || !m->measure) {
        set_error("tt_integrate_p1: bad mesh");
        return TT_ERR_INVALID_PARAMETER;
    }
    const int k = m->dim + 1;
    LocalMass w;
    for (int i = 0; i < 16; ++i) w.m[i] = 0.0;
    // w = rule.points^T @ rule.weights for the degree-2 rule (fem.py:158-160)
    if (k == 3) {
        const double P[3][3] = {{2.0 / 3, 1.0 / 6, 1.0 / 6}, {1.0 / 6, 2.0 / 3, 1.0 / 6}, {1.0 / 6, 1.0 / 6, 2.0 / 3}};
        for (int a = 0; a < 3; ++a) {
            double s = 0.0;
            for (int q = 0; q < 3; ++q) s += P[q][a] * (1.0 / 3);
            w.m[a] = s;
        }
    } else {
        for (int a = 0; a < 4; ++a) w.m[a] = 0.25;
    }
    auto s = as_stream(stream);
    const int nparts = sm_count() * 2;
    double* part = nullptr;
    int st = cuda_status(cudaMallocAsync((void**)&part, sizeof(double) * nparts, s), "integrate alloc");
    if (st) return st;
    integrate_kernel<<<nparts, 256, 0, s>>>(m->n_elems, k, m->elems, m->measure, coeffs, w, part);
    sum_parts_kernel<<<1, 32, 0, s>>>(nparts, part, out);
    st = launch_check("integrate kernels");
    cudaFreeAsync(part, s);
    return st;
}

extern "C" int tt_csr_to_ell(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, int width,
                             int32_t* ell_cols, double* ell_vals, double* diag, int32_t* status,
                             void* stream) {
    if (n < 1 || (width != 16 && width != 8)) {
        set_error("tt_csr_to_ell: width must be 8 or 16");
        return TT_ERR_INVALID_PARAMETER;
    }
    csr_to_ell_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, rp, ci, v, width, ell_cols, ell_vals,
                                                                        diag, status);
    return launch_check("csr_to_ell_kernel");
}

static int blocks_per_sm(const void* fn, int block, size_t smem) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, block, smem);
    return per < 1 ? 1 : per;
}

static bool ell_args(EllArgs& a, int64_t n, int width, const int32_t* ell_cols, const double* ell_vals,
                     const double* diag, const double* b, double tol, int64_t maxiter, double* x,
                     double* best_x, double* work, tt_pcg_result_t* result, const char* who) {
    if (n < 1 || maxiter < 0 || (width != 8 && width != 16)) {
        set_error("%s: bad size or width (8 | 16)", who);
        return false;
    }
    a.n = n; a.ec = ell_cols; a.ev = ell_vals; a.diag = diag; a.b = b; a.tol = tol; a.maxiter = maxiter;
    a.x = x; a.best_x = best_x;
    a.r = work; a.z = work + n; a.p0 = work + 2 * n; a.p1 = work + 3 * n; a.ap = work + 4 * n;
    a.dinv = work + 5 * n;
    a.part = work + 6 * n;
    a.res = result;
    a.slab_rows = 0;
    return true;
}

extern "C" int tt_pcg_ell(int64_t n, int width, const int32_t* ell_cols, const double* ell_vals,
                          const double* diag, const double* b, double tol, int64_t maxiter, double* x,
                          double* best_x, double* work, tt_pcg_result_t* result, void* stream) {
    EllArgs a;
    if (!ell_args(a, n, width, ell_cols, ell_vals, diag, b, tol, maxiter, x, best_x, work, result, "tt_pcg_ell"))
        return TT_ERR_INVALID_PARAMETER;
    // SpMV shape: W/8 lanes per row, every block a contiguous row range.  Measured on the C2
    // mass matrix (175,616 rows, 23 iterations): 2 lanes + contiguous 0.357 ms, 4 lanes +
    // contiguous 0.373 ms, 4 lanes + grid-stride 0.377 ms, 2 lanes + grid-stride 0.404 ms.
    const int lpr = width / 8;
    const void* fn = width == 8 ? (const void*)pcg_ell_kernel<512, 2, 8, false>
                                : (const void*)pcg_ell_kernel<512, 2, 16, false>;
    static const int per8 = blocks_per_sm((const void*)pcg_ell_kernel<512, 2, 8, false>, 512, 0);
    static const int per16 = blocks_per_sm((const void*)pcg_ell_kernel<512, 2, 16, false>, 512, 0);
    const int per_sm = width == 8 ? per8 : per16;
    int64_t maxb = (int64_t)sm_count() * per_sm;
    int64_t need = (n * lpr + 511) / 512;
    if (need < 1) need = 1;
    int blocks = (int)(need < maxb ? need : maxb);
    if (blocks > 148 * 32) blocks = 148 * 32;
    void* args[] = {&a};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(512), args, 0, as_stream(stream));
    return cuda_status(e, "pcg_ell_kernel (cooperative launch)");
}

extern "C" int tt_pcg_ell_slab(int64_t n, int width, const int32_t* ell_cols, const double* ell_vals,
                               const double* diag, const double* b, double tol, int64_t maxiter, double* x,
                               double* best_x, double* work, tt_pcg_result_t* result, void* stream) {
    EllArgs a;
    if (!ell_args(a, n, width, ell_cols, ell_vals, diag, b, tol, maxiter, x, best_x, work, result,
                  "tt_pcg_ell_slab"))
        return TT_ERR_INVALID_PARAMETER;
    const int lpr = width / 8;  // lanes per row = 80-byte chunks per row
    const void* fn = width == 8 ? (const void*)pcg_ell_kernel<512, 2, 8, true>
                                : (const void*)pcg_ell_kernel<512, 2, 16, true>;
    int dev = 0, max_optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int sms = sm_count();
    // rows that must be slab-resident for the slab to pay (1/2): the rest of a block's rows
    // stream from L2/HBM as in tt_pcg_ell, with the L1 the slab took.  Measured per 3-D
    // solve, slab vs L2 kernel: 59 % on chip (357,911 rows) 0.565 vs 0.691 ms; 40 %
    // (531,441) 1.20 vs 1.04; 28 % (753,571) 1.83 vs 1.25; C1 (2-D, 85 %) 0.36 vs 0.43
    constexpr double min_frac = 0.5;
    // 2 blocks per SM (the 2 x 512 shape of tt_pcg_ell), else 1 with twice the rows.  With
    // 2 per SM the block count and row ranges are tt_pcg_ell's, so the partial sums -- and
    // the iterates -- are bitwise the same
    const int64_t need = (n * lpr + 511) / 512;
    for (int bps = 2; bps >= 1; --bps) {
        const int64_t nb = need < (int64_t)sms * bps ? need : (int64_t)sms * bps;
        const int64_t rpb = (n + nb - 1) / nb;
        const int64_t per_row = 80 * lpr;
        // per-SM shared memory: 228 KB less 1 KB per block reserved, less the static part
        const int64_t avail = (int64_t)(bps == 2 ? (228 * 1024) / 2 - 1024 : max_optin) - (int64_t)sizeof(double) * 96;
        const int64_t cap = avail / per_row;
        const int64_t rows = rpb < cap ? rpb : cap;
        if (rows < 1 || (rows < rpb && rows < min_frac * rpb)) continue;
        const int64_t smem = rows * per_row;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 512, (size_t)smem);
        if (per_sm < bps) continue;
        a.slab_rows = rows;
        void* args[] = {&a};
        cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)nb), dim3(512), args, (size_t)smem,
                                                    as_stream(stream));
        return cuda_status(e, "pcg_ell_kernel (slab, cooperative launch)");
    }
    set_error("tt_pcg_ell_slab: too few of the %lld rows fit in shared memory", (long long)n);
    return TT_ERR_CAPACITY;
}

// launch shape of the pipelined kernels (threads per block, blocks per SM)
#ifndef TT_PIPE_BLOCK
#define TT_PIPE_BLOCK 512
#endif
#ifndef TT_PIPE_MINB
#define TT_PIPE_MINB 1
#endif
constexpr int kPB = TT_PIPE_BLOCK, kPM = TT_PIPE_MINB;

static bool pipe_args(PipeArgs& a, int64_t n, int width, const int32_t* ell_cols, const double* ell_vals,
                      const double* diag, const double* b, double tol, int64_t maxiter, double* x,
                      double* best_x, double* work, tt_pcg_result_t* result, const char* who) {
    if (n < 1 || maxiter < 0 || (width != 8 && width != 16)) {
        set_error("%s: bad size or width (8 | 16)", who);
        return false;
    }
    a.n = n; a.ec = ell_cols; a.ev = ell_vals; a.diag = diag; a.b = b; a.tol = tol; a.maxiter = maxiter;
    a.x = x; a.best_x = best_x;
    double* v[10];
    for (int k = 0; k < 10; ++k) v[k] = work + k * n;
    a.r = v[0]; a.u = v[1]; a.w = v[2]; a.z = v[3]; a.q = v[4]; a.s = v[5]; a.p = v[6];
    a.m0 = v[7]; a.m1 = v[8]; a.dinv = v[9];
    a.part = work + 10 * n;
    a.res = result;
    a.slab_rows = 0;
    return true;
}

// The pipelined recurrence with the rows on chip (1 grid barrier per iteration).  Measured per
// solve (scripts/pcg_ab.py): C2 mass matrix 0.329 -> 0.262 ms (23 iterations), C1 0.329 ->
// 0.316 ms; one 512-thread block per SM (the recurrence needs ~110 registers; two blocks
// of 512 spill, 0.357 ms).  Streaming the rows from L2/HBM (C4) it is slower than the
// textbook kernel (2.9 vs 2.4 ms: ten vectors per row instead of six), so tt_pcg_ell keeps
// the textbook recurrence.
extern "C" int tt_pcg_ell_slab_pipelined(int64_t n, int width, const int32_t* ell_cols, const double* ell_vals,
                               const double* diag, const double* b, double tol, int64_t maxiter, double* x,
                               double* best_x, double* work, tt_pcg_result_t* result, void* stream) {
    PipeArgs a;
    if (!pipe_args(a, n, width, ell_cols, ell_vals, diag, b, tol, maxiter, x, best_x, work, result,
                   "tt_pcg_ell_slab_pipelined"))
        return TT_ERR_INVALID_PARAMETER;
    const int cpr = width / 8;  // 80-byte slab chunks per row
    const void* fn = width == 8 ? (const void*)pcg_pipe_kernel<kPB, kPM, 8, true>
                                : (const void*)pcg_pipe_kernel<kPB, kPM, 16, true>;
    int dev = 0, max_optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int sms = sm_count();
    // rows that must be slab-resident for the slab to pay (1/2): the rest of a block's rows
    // stream from L2/HBM as in tt_pcg_ell, with the L1 the slab took.  Measured per 3-D
    // solve, slab vs L2 kernel: 59 % on chip (357,911 rows) 0.565 vs 0.691 ms; 40 %
    // (531,441) 1.20 vs 1.04; 28 % (753,571) 1.83 vs 1.25; C1 (2-D, 85 %) 0.36 vs 0.43
    constexpr double min_frac = 0.5;
    // kPM blocks per SM (one 512-thread block: the recurrence needs ~128 registers), blocks of
    // at least kPB / 2 rows (one lane per row), at most one wave
    const int64_t need = (2 * n + kPB - 1) / kPB;
    for (int bps = kPM; bps >= 1; --bps) {
        const int64_t nb = need < (int64_t)sms * bps ? need : (int64_t)sms * bps;
        const int64_t rpb = (n + nb - 1) / nb;
        const int64_t per_row = 80 * cpr;
        // per-SM shared memory: 228 KB less 1 KB per block reserved, less the static part
        const int64_t avail = (int64_t)(bps > 1 ? (228 * 1024) / bps - 1024 : max_optin) - (int64_t)sizeof(double) * 96 - 16;
        const int64_t cap = avail / per_row;
        const int64_t rows = rpb < cap ? rpb : cap;
        if (rows < 1 || (rows < rpb && rows < min_frac * rpb)) continue;
        const int64_t smem = rows * per_row;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPB, (size_t)smem);
        if (per_sm < bps) continue;
        a.slab_rows = rows;
        void* args[] = {&a};
        cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)nb), dim3(kPB), args, (size_t)smem,
                                                    as_stream(stream));
        return cuda_status(e, "pcg_pipe_kernel (slab, cooperative launch)");
    }
    set_error("tt_pcg_ell_slab_pipelined: too few of the %lld rows fit in shared memory", (long long)n);
    return TT_ERR_CAPACITY;
}

#ifdef TT_PCG_TRACE
extern "C" int tt_debug_pcg_trace(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_pcg_trace, sizeof(g_pcg_trace));
}
#endif
