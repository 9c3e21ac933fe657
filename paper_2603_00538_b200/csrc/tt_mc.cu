// Fused Monte-Carlo load assembly (montecarlo.py:110-147) for P1 simplices, d = 2, 3.
//
// One kernel does plan -> point map -> black-box source query -> f*lambda accumulation:
//   * a lane GROUP of G lanes (G in {8, 16, 32}) owns one target element; its lanes
//     stride over the element's N samples, so the 32 lanes of a warp query points of
//     one (or a few spatially adjacent) elements: the source-side candidate lists and
//     locate records they touch are shared and come from L1 (broadcast loads);
//   * per-lane k-vector accumulators in registers, then a G-lane xor-shuffle tree
//     (warp-aggregated reduction) -> one write of contrib[e, 0..k) per element, or one
//     atomicAdd per (element, vertex) into b when no contribution buffer is given;
//   * nothing per-sample touches HBM: shared-plan lambdas are an L1-resident (N, k)
//     table, Philox plans are generated in-register, and the source field is either an
//     analytic postfix program (kernel parameter space) or a P1 nodal field located
//     through the uniform grid in-register (locate + snap + gather).
// The element contribution is (sum_j f_j lambda_j) / (N * (1/|T|)) -- the reference's
// (f / (n p)) @ lam with the per-element constant factored out (montecarlo.py:128-131).
#include <cub/cub.cuh>
#include "tt_common.cuh"
#include "tt_philox.cuh"

namespace tt {

struct SrcDev {
    int kind;
    int outside;
    GridDev grid;
    const int32_t* __restrict__ src_elems;
    const double* __restrict__ coeffs;
    const double* __restrict__ values;
    const int32_t* __restrict__ cached;
    const int32_t* __restrict__ seeds;
    const double* __restrict__ ecoef;
    const double* __restrict__ egrad;
    const double* __restrict__ density;  // importance weights p (e_hi-e_lo, N), or NULL = 1/|T|
};

template <int D>
__device__ __forceinline__ double eval_expr(const tt_expr_t& p, const double* x) {
    double st[TT_EXPR_MAX_STACK];
    int sp = 0;
    for (int i = 0; i < p.n_ops; ++i) {
        const int op = p.ops[i];
        switch (op) {
            case TT_OP_CONST: st[sp++] = p.consts[i]; break;
            case TT_OP_X: st[sp++] = x[0]; break;
            case TT_OP_Y: st[sp++] = x[1]; break;
            case TT_OP_Z: st[sp++] = (D == 3) ? x[D - 1] : 0.0; break;
            case TT_OP_ADD: --sp; st[sp - 1] = st[sp - 1] + st[sp]; break;
            case TT_OP_SUB: --sp; st[sp - 1] = st[sp - 1] - st[sp]; break;
            case TT_OP_MUL: --sp; st[sp - 1] = st[sp - 1] * st[sp]; break;
            case TT_OP_DIV: --sp; st[sp - 1] = st[sp - 1] / st[sp]; break;
            case TT_OP_POW: --sp; st[sp - 1] = pow(st[sp - 1], st[sp]); break;
            case TT_OP_SQUARE: st[sp - 1] = st[sp - 1] * st[sp - 1]; break;
            case TT_OP_NEG: st[sp - 1] = -st[sp - 1]; break;
            case TT_OP_SIN: st[sp - 1] = sin(st[sp - 1]); break;
            case TT_OP_COS: st[sp - 1] = cos(st[sp - 1]); break;
            case TT_OP_EXP: st[sp - 1] = exp(st[sp - 1]); break;
            case TT_OP_SQRT: st[sp - 1] = sqrt(st[sp - 1]); break;
            case TT_OP_LOG: st[sp - 1] = log(st[sp - 1]); break;
            case TT_OP_TAN: st[sp - 1] = tan(st[sp - 1]); break;
            case TT_OP_ABS: st[sp - 1] = fabs(st[sp - 1]); break;
            default: break;
        }
    }
    return sp > 0 ? st[0] : 0.0;
}

// P1 evaluation sum_i c_i lambda_i at source element e: from the packed per-element
// coefficient record when present (one aligned 32 B load), else conn + coeff gathers.
template <int D>
__device__ __forceinline__ double p1_eval(const SrcDev& s, int e, const double* l) {
    constexpr int K = D + 1;
    double c[K];
    if (s.ecoef) {
        const double2* q = reinterpret_cast<const double2*>(s.ecoef + (int64_t)e * 4);
        const double2 a = __ldg(q), b = __ldg(q + 1);
        c[0] = a.x; c[1] = a.y; c[2] = b.x;
        if constexpr (D == 3) c[3] = b.y;
    } else {
        const int32_t* conn = s.src_elems + (int64_t)e * K;
#pragma unroll
        for (int i = 0; i < K; ++i) c[i] = __ldg(s.coeffs + __ldg(conn + i));
    }
    double f = mul(c[0], l[0]);
#pragma unroll
    for (int i = 1; i < K; ++i) f = add(f, mul(c[i], l[i]));
    return f;
}

// MeshBackedField.__call__ (montecarlo.py:49-65) + eval_in_elements (fem.py:36-38)
template <int D>
__device__ __forceinline__ double eval_mesh(const SrcDev& s, const double* x, int& flags, int& guess) {
    constexpr int K = D + 1;
    double l[K];
    int e = (s.grid.walk && guess >= 0) ? locate_walk<D>(s.grid, x, 1e-12, guess, l)
                                        : locate_point<D>(s.grid, x, 1e-12, l);
    if (e >= 0) guess = e;
    if (e < 0) {
        if (s.outside == TT_OUTSIDE_STRICT) {
            flags |= TT_FLAG_OUTSIDE_STRICT;
            return 0.0;
        }
        const SnapOut<D> sn = snap_point<D>(s.grid, x[0], x[1], D == 3 ? x[D - 1] : 0.0);
        e = sn.e;
#pragma unroll
        for (int i = 0; i < K; ++i) l[i] = sn.l[i];
    }
    return p1_eval<D>(s, e, l);
}

// cached source element: lambda_s for ALL samples clipped >= 0 and renormalised
// (transfer.py:84-87), then the P1 gather
template <int D>
__device__ __forceinline__ double eval_cached(const SrcDev& s, const double* x, int e) {
    constexpr int K = D + 1;
    double l[K];
    snap_lambda<D>(s.grid, e, x, l);
    return p1_eval<D>(s, e, l);
}

template <int D, int SRC>
__device__ __forceinline__ double eval_source(const SrcDev& s, const tt_expr_t& expr,
                                              const double* x, int64_t vidx, int& flags,
                                              int& guess) {
    if constexpr (SRC == TT_SRC_EXPR) return eval_expr<D>(expr, x);
    else if constexpr (SRC == TT_SRC_MESH) return eval_mesh<D>(s, x, flags, guess);
    else if constexpr (SRC == TT_SRC_CACHED) return eval_cached<D>(s, x, __ldg(s.cached + vidx));
    else return __ldg(s.values + vidx);
}

template <int D>
__device__ __forceinline__ void philox_lambda(uint64_t seed, int64_t e, int64_t j, double* lam) {
    double xi[3];
    philox_uniforms(seed, (uint64_t)e, (uint64_t)j, xi);
    if constexpr (D == 2) {
        double r = __dsqrt_rn(xi[0]);
        lam[0] = sub(1.0, r);
        lam[1] = mul(r, sub(1.0, xi[1]));
        lam[2] = mul(r, xi[1]);
    } else {
        double r = cbrt(xi[0]);
        double q = __dsqrt_rn(xi[1]);
        double rq = mul(r, q);
        lam[0] = sub(1.0, r);
        lam[1] = mul(r, sub(1.0, q));
        lam[2] = mul(rq, sub(1.0, xi[2]));
        lam[3] = mul(rq, xi[2]);
    }
}

struct TargetDev {
    const double* __restrict__ nodes;
    const int32_t* __restrict__ elems;
    const double* __restrict__ measure;
    const int32_t* __restrict__ gid;  // optional global element ids (Philox counters)
};

// Philox stream counter of element e: its global id (a rank's partition mesh numbers its
// elements locally; tt_mesh_t.gid maps them back), so streams are partition independent
__device__ __forceinline__ int64_t stream_id(const int32_t* __restrict__ gid, int64_t e) {
    return gid ? (int64_t)__ldg(gid + e) : e;
}

struct PlanDev {
    int64_t n;
    const double* __restrict__ lam;
    uint64_t seed;
    const int32_t* __restrict__ order;  // fused SLOT kernel: lam is the plan's table in this
                                        // order (lam_walk); ids are written back at order[j]
    const double* __restrict__ lam_walk;
};

template <int D>
__device__ __forceinline__ void load_elem(const TargetDev& t, int64_t e, double (*v)[D]) {
    constexpr int K = D + 1;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        int64_t n = __ldg(t.elems + e * K + i);
#pragma unroll
        for (int c = 0; c < D; ++c) v[i][c] = __ldg(t.nodes + n * D + c);
    }
}

template <int D, int PLAN, int SRC, int G>
__global__ void __launch_bounds__(256) mc_load_kernel(TargetDev t, int64_t e_lo, int64_t e_hi,
                                                      PlanDev plan, SrcDev src,
                                                      const __grid_constant__ tt_expr_t expr,
                                                      double* __restrict__ contrib, int64_t cld,
                                                      double* __restrict__ b,
                                                      int32_t* __restrict__ status) {
    constexpr int K = D + 1;
    constexpr int EPW = 32 / G;  // elements per warp tile
    const int lane = threadIdx.x & 31;
    const int sub_lane = lane % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t n_el = e_hi - e_lo;
    const int64_t N = plan.n;
    int flags = 0;

    for (int64_t tile = warp; tile * EPW < n_el; tile += nwarps) {
        const int64_t le = tile * EPW + lane / G;  // local element index
        const bool active = le < n_el;
        const int64_t e = e_lo + le;
        double acc[K];
#pragma unroll
        for (int i = 0; i < K; ++i) acc[i] = 0.0;
        if (active) {
            double v[K][D];
            load_elem<D>(t, e, v);
            int guess = -1;
            if constexpr (SRC == TT_SRC_MESH)
                if (src.seeds) guess = __ldg(src.seeds + e * kSeeds);
            for (int64_t j = sub_lane; j < N; j += G) {
                double lam[K];
                if constexpr (PLAN == TT_PLAN_SHARED) {
#pragma unroll
                    for (int i = 0; i < K; ++i) lam[i] = __ldg(plan.lam + j * K + i);
                } else {
                    philox_lambda<D>(plan.seed, stream_id(t.gid, e), j, lam);
                }
                double x[D];
                map_point<D>(lam, v, x);
                double f = eval_source<D, SRC>(src, expr, x, le * N + j, flags, guess);
                if (!isfinite(f)) flags |= TT_FLAG_NONFINITE;
                if (src.density) {
                    // importance-weighted estimator: f / (N p) per sample (montecarlo.py:128-131)
                    const double p = __ldg(src.density + le * N + j);
                    if (p <= 0.0) flags |= TT_FLAG_INVALID_DENSITY;
                    f = f / ((double)N * p);
                }
#pragma unroll
                for (int i = 0; i < K; ++i) acc[i] = fma(f, lam[i], acc[i]);
            }
        }
        // G-lane xor tree (groups are aligned power-of-two lane ranges)
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1)
#pragma unroll
            for (int i = 0; i < K; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
        if (active && sub_lane == 0) {
            // (sum f lam) / (N p), p = 1/|T|  (montecarlo.py:128-131, :135-141); with a
            // density the weights were applied per sample
            const double q = src.density ? 1.0 : (double)N * (1.0 / __ldg(t.measure + e));
            if (contrib) {
#pragma unroll
                for (int i = 0; i < K; ++i) contrib[cld ? i * cld + le : le * K + i] = acc[i] / q;
            } else {
#pragma unroll
                for (int i = 0; i < K; ++i) atomicAdd(b + __ldg(t.elems + e * K + i), acc[i] / q);
            }
        }
    }
    if (flags) atomicOr(status, flags);
}

template <int D, int PLAN>
__device__ __forceinline__ void plan_lambda(const PlanDev& plan, const int32_t* gid, int64_t e, int64_t j,
                                            double* lam) {
    constexpr int K = D + 1;
    if constexpr (PLAN == TT_PLAN_SHARED) {
        if constexpr (D == 3) {
            const double2* q = reinterpret_cast<const double2*>(plan.lam + j * 4);
            const double2 a = __ldg(q), b = __ldg(q + 1);
            lam[0] = a.x; lam[1] = a.y; lam[2] = b.x; lam[3] = b.y;
        } else {
#pragma unroll
            for (int i = 0; i < K; ++i) lam[i] = __ldg(plan.lam + j * K + i);
        }
    } else {
        philox_lambda<D>(plan.seed, stream_id(gid, e), j, lam);
    }
}

#ifdef TT_MC_STATS
// instrumentation build only (-DTT_MC_STATS): loop iterations, busy lanes, samples, walk
// steps, exact fallbacks of mc_mesh_kernel
__device__ unsigned long long g_mc_stats[8];
#define TT_STAT(i, v) atomicAdd(&g_mc_stats[i], (unsigned long long)(v))
#else
#define TT_STAT(i, v) ((void)0)
#endif

constexpr int kSlotCap = 4096;  // per-block seed-slot table capacity (samples)

// Per-element (Philox) plans have no slot table: a lookup table of the nearest anchor over a
// grid of barycentric space (3-D: 16^3 cells of (l0, l1, l2); 2-D: 64^2 of (l0, l1)), built
// once per process for 16 and for kSeeds anchors, gives each sample a near-nearest walk
// anchor for one L1-resident byte load (the seed is only a walk start: its choice never
// changes a result).
constexpr int kAnchorTab = 4096;
__device__ uint8_t g_anchor_tab[2][2][kAnchorTab];   // [dim - 2][all anchors][cell]

template <int D>
__global__ void anchor_tab_kernel(int n_anchors, uint8_t* __restrict__ tab) {
    constexpr int K = D + 1;
    constexpr int Q = D == 3 ? 16 : 64;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= kAnchorTab) return;
    double l[K];
    if constexpr (D == 3) {
        l[0] = ((c / (Q * Q)) + 0.5) / Q; l[1] = (((c / Q) % Q) + 0.5) / Q; l[2] = ((c % Q) + 0.5) / Q;
    } else {
        l[0] = ((c / Q) + 0.5) / Q; l[1] = ((c % Q) + 0.5) / Q;
    }
    double rest = 1.0;
    for (int a = 0; a < D; ++a) rest -= l[a];
    l[D] = rest;
    int best = 0;
    double dbest = 1e300;
    for (int m = 0; m < n_anchors; ++m) {
        double d = 0.0;
        for (int a = 0; a <= D; ++a) { const double u = l[a] - anchor<D>(m, a); d += u * u; }
        if (d < dbest) { dbest = d; best = m; }
    }
    tab[c] = (uint8_t)best;
}

template <int D>
__device__ __forceinline__ int seed_slot_tab(const double* lam, int all) {
    constexpr int Q = D == 3 ? 16 : 64;
    const auto q = [](double v) { int i = (int)(v * Q); return i < 0 ? 0 : (i > Q - 1 ? Q - 1 : i); };
    const int c = D == 3 ? (q(lam[0]) * Q + q(lam[1])) * Q + q(lam[2]) : q(lam[0]) * Q + q(lam[1]);
    return g_anchor_tab[D - 2][all][c];
}

static int anchor_tables_ready(cudaStream_t st) {
    static unsigned long long done = 0;   // per device (bit = device ordinal)
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done & bit) return TT_OK;
    uint8_t* tab = nullptr;
    int rc = cuda_status(cudaGetSymbolAddress((void**)&tab, g_anchor_tab), "anchor table");
    if (rc) return rc;
    anchor_tab_kernel<2><<<kAnchorTab / 256, 256, 0, st>>>(16, tab);
    anchor_tab_kernel<2><<<kAnchorTab / 256, 256, 0, st>>>(kSeeds, tab + kAnchorTab);
    anchor_tab_kernel<3><<<kAnchorTab / 256, 256, 0, st>>>(16, tab + 2 * kAnchorTab);
    anchor_tab_kernel<3><<<kAnchorTab / 256, 256, 0, st>>>(kSeeds, tab + 3 * kAnchorTab);
    rc = launch_check("anchor_tab_kernel");
    if (!rc) done |= bit;
    return rc;
}

// With a per-block slot table (shared plans): the nearest of all kSeeds anchors in
// barycentric space (66.7 % of samples lie in its source element at C2 vs 56.5 % for the
// closed-form rule above, scripts/seed_anchors.py)
template <int D>
__device__ __forceinline__ int seed_slot_nearest(const double* lam, int n_anchors) {
    int best = 0;
    double dbest = 1e300;
    for (int m = 0; m < n_anchors; ++m) {
        double d = 0.0;
#pragma unroll
        for (int a = 0; a <= D; ++a) {
            const double u = lam[a] - anchor<D>(m, a);
            d = fma(u, u, d);
        }
        if (d < dbest) { dbest = d; best = m; }
    }
    return best;
}

// Mesh-backed source, flattened walk: each loop iteration performs exactly ONE facet-walk
// step for every busy lane, and idle lanes immediately take the element's next unprocessed
// sample (ballot + popc inside the G-lane group).  SIMT lanes stay busy regardless of how
// many steps individual samples need; the assignment is a deterministic function of the
// data, so results are bitwise reproducible.  Identical ids/lambdas as the reference scan
// (certified walk, see locate_walk in tt_common.cuh).
//
// Launch shape: 128-thread blocks, 5 resident per SM at <= 96 registers,
// each element's vertices and walk seeds in shared memory, one wave of blocks (a
// persistent tile loop).  Walk steps read the compact 80 B float record (wrec) and
// evaluate f from the element's gradient record (egrad), loaded speculatively with it.
//   SLOT  (shared plans, N <= kSlotCap): per-block table of each sample's nearest walk
//         anchor (N bytes of dynamic shared memory), built once per block.
//   DEFER (pairs whose seeds saw outside anchors): an outside sample's nearest-element
//         search is parked and run warp-cooperatively at the end of the tile.
#ifndef TT_MC_MINB
#define TT_MC_MINB 5
#endif
constexpr int kMcBlock = 128;
constexpr int kMcMinBlocks = TT_MC_MINB;

template <int D, int PLAN, int G, bool SLOT, bool DEFER>
__global__ void __launch_bounds__(kMcBlock, kMcMinBlocks) mc_mesh_kernel(TargetDev t, int64_t e_lo, int64_t e_hi,
                                                      PlanDev plan, SrcDev src,
                                                      double* __restrict__ contrib, int64_t cld,
                                                      double* __restrict__ b,
                                                      int32_t* __restrict__ ids_out,
                                                      int32_t* __restrict__ status) {
    constexpr int K = D + 1;
    constexpr int EPW = 32 / G;
    constexpr int NW = kMcBlock / 32;
    constexpr double EPS = 1e-12;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const unsigned lt = (1u << lane) - 1u;
    const int sub_lane = lane % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t n_el = e_hi - e_lo;
    const int64_t N = plan.n;
    const GridDev& g = src.grid;
    const bool walk = g.walk && src.seeds && g.wrec;
    int flags = 0;
    constexpr bool USE_SLOT = SLOT && PLAN == TT_PLAN_SHARED;
    const int n_anchors = G <= 2 ? 16 : seeds_used(plan.n);   // the seed table's first columns
    // SLOT: each sample's nearest walk anchor.  With plan.order the launch passes the plan's
    // table in that order (tt_plan_walk_order: grouped by nearest anchor, so a group's lanes
    // start their walks from the same seed element); sample j here is plan sample order[j]
    extern __shared__ int8_t s_slot[];  // N bytes (launch: dynamic shared memory)
    if constexpr (USE_SLOT) {
        for (int64_t j = threadIdx.x; j < N; j += kMcBlock) {
            double lj[K];
            plan_lambda<D, PLAN>(plan, t.gid, 0, j, lj);
            s_slot[j] = (int8_t)seed_slot_nearest<D>(lj, n_anchors);
        }
        __syncthreads();
    }
    // vertex rows of VS doubles read as double2 (LDS.128): VS = 2 (mod 4) puts the 16-byte
    // reads of a warp's (up to 8) groups on distinct bank quads; seed rows padded to 17 ints
    constexpr int VS = D == 3 ? 14 : 6;
    __shared__ __align__(16) double s_v[NW][EPW][VS];
    // seed rows padded to an odd length; 2-lane groups (N < 32) use the first 16 anchors only
    constexpr int SROW = G <= 2 ? 17 : kSeeds + 1;
    __shared__ int s_seed[NW][EPW][SROW];
    const int wib = threadIdx.x >> 5, gib = lane / G;

    for (int64_t tile = warp; tile * EPW < n_el; tile += nwarps) {
        const int64_t le = tile * EPW + lane / G;
        const bool active = le < n_el;
        const int64_t e = e_lo + le;
        double acc[K];
#pragma unroll
        for (int i = 0; i < K; ++i) acc[i] = 0.0;
        __syncwarp();
        if (active) {
            for (int q = sub_lane; q < K * D; q += G)
                s_v[wib][gib][q] = __ldg(t.nodes + (int64_t)__ldg(t.elems + e * K + q / D) * D + q % D);
            if (walk)
                for (int q = sub_lane; q < n_anchors; q += G)
                    s_seed[wib][gib][q] = __ldg(src.seeds + e * kSeeds + q);
        }
        __syncwarp();
        const auto vertices = [&](double (*vv)[D]) {
            const double2* row = reinterpret_cast<const double2*>(s_v[wib][gib]);
#pragma unroll
            for (int q = 0; q < K * D / 2; ++q) {
                const double2 u = row[q];
                vv[(2 * q) / D][(2 * q) % D] = u.x;
                vv[(2 * q + 1) / D][(2 * q + 1) % D] = u.y;
            }
        };
        int next = 0;
        int jcur = 0;
        int pend_j = -1;  // DEFER: this lane's outside sample whose snap runs at tile end
        bool busy = false;
        double x[D], lam[K];
        int cur = -1, steps = 0;
        while (true) {
            const bool want = active && !busy;
            const unsigned m = __ballot_sync(FULL, want) & gmask;
            if (want) {
                const int j = next + __popc(m & lt);
                if (j < N) {
                    plan_lambda<D, PLAN>(plan, t.gid, e, j, lam);
                    double vv[K][D];
                    vertices(vv);
                    map_point_fma<D>(lam, vv, x);
                    cur = -1;
                    if (walk) {
                        int slot;
                        if constexpr (USE_SLOT) slot = s_slot[j];
                        else slot = seed_slot_tab<D>(lam, n_anchors > 16);   // Philox: lookup table
                        cur = s_seed[wib][gib][slot];
                    }
                    steps = 0;
                    jcur = j;
                    busy = true;
                }
            }
            next += __popc(m);
            if (!__any_sync(FULL, busy)) break;
#ifdef TT_MC_STATS
            {
                const unsigned bm = __ballot_sync(FULL, busy);
                if (lane == 0) { TT_STAT(0, 1); TT_STAT(1, __popc(bm)); }
            }
#endif
            if (!busy) continue;
            double l[K];
            int hit = -1;
            int fb = -1;  // element whose float test fell in its uncertainty band
            bool done = false;
            bool fw_hit = false;
            double fw_f = 0.0;
            if (cur >= 0 && steps < 12) {
                // compact float walk step: exact ids via a margin that bounds the float
                // evaluation error (tt_grid.cu walk_prep_kernel); f from the element's
                // gradient record: f = c_last + g . (x - o), accurate to a few ulps
                WRec<D> w;
                load_wrec<D>(g.wrec, cur, w);
                double2 pc0 = make_double2(0.0, 0.0), pc1 = make_double2(0.0, 0.0);
                if (src.egrad) {  // speculative: the gradient record of the element tested
                    const double2* q = reinterpret_cast<const double2*>(src.egrad + (int64_t)cur * 4);
                    pc0 = __ldg(q);
                    pc1 = __ldg(q + 1);
                }
                double r[D];
                float rf[D];
#pragma unroll
                for (int c = 0; c < D; ++c) { r[c] = x[c] - w.o[c]; rf[c] = __double2float_rn(r[c]); }
                float lf[K];
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    float a = w.b[i][0] * rf[0];
#pragma unroll
                    for (int c = 1; c < D; ++c) a = fmaf(w.b[i][c], rf[c], a);
                    lf[i] = a;
                }
                float last = 1.0f - lf[0] - lf[1];
                if constexpr (D == 3) last -= lf[2];
                lf[D] = last;
                int imin = 0;
                float lmin = lf[0];
#pragma unroll
                for (int i = 1; i <= D; ++i)
                    if (lf[i] < lmin) { lmin = lf[i]; imin = i; }
                if (lmin >= w.tau) {
                    hit = cur;
                    done = true;
                    fw_hit = true;
                    const double gv[4] = {pc0.x, pc0.y, pc1.x, pc1.y};
                    double f = gv[D];
#pragma unroll
                    for (int c = 0; c < D; ++c) f = fma(gv[c], r[c], f);
                    fw_f = f;
                } else if (lmin > -w.tau) {
                    fb = cur;  // within the uncertainty band of a facet: exact double walk
                    cur = -1;
                } else {
                    int nb = w.nbr[0];
#pragma unroll
                    for (int i = 1; i <= D; ++i)
                        if (imin == i) nb = w.nbr[i];
                    cur = nb;
                    ++steps;
                    TT_STAT(3, 1);
                }
            } else {
                cur = -1;
            }
            if (!done && cur < 0) {
                // exact localisation (rare): the walk mapped the point with FMA, so recompute
                // it in the reference's op order first (montecarlo.py:123-124); then the
                // double certified walk from the band element (one diverged lane, ~1
                // dependent record load) or the reference cell scan
                {
                    double vv[K][D];
                    vertices(vv);
                    map_point<D>(lam, vv, x);
                }
                hit = fb >= 0 ? locate_walk<D>(g, x, EPS, fb, l) : locate_point<D>(g, x, EPS, l);
                bool deferred = false;
                if (hit < 0) {
                    if (src.outside == TT_OUTSIDE_STRICT) {
                        flags |= TT_FLAG_OUTSIDE_STRICT;
                    } else if (DEFER && ids_out == nullptr && pend_j < 0) {
                        // the nearest-element ring search runs at the end of the tile with
                        // the whole warp (nearest_element_warp) instead of on this one lane
                        pend_j = jcur;
                        deferred = true;
                        flags |= TT_FLAG_SNAPPED;
                        TT_STAT(5, 1);
                    } else {
                        flags |= TT_FLAG_SNAPPED;
                        TT_STAT(5, 1);
                        const SnapOut<D> sn = snap_point<D>(g, x[0], x[1], D == 3 ? x[D - 1] : 0.0);
                        hit = sn.e;
#pragma unroll
                        for (int i = 0; i < K; ++i) l[i] = sn.l[i];
                    }
                }
                done = true;
                if (deferred) {
                    busy = false;  // the sample's contribution is added at tile end
                    continue;
                }
            }
            if (done) {
                TT_STAT(2, 1);
                if (!fw_hit) TT_STAT(4, 1);
                if (ids_out) ids_out[le * N + (plan.order ? plan.order[jcur] : jcur)] = hit;
                double f = 0.0;
                if (fw_hit) f = fw_f;
                else if (hit >= 0 && (contrib || b)) f = p1_eval<D>(src, hit, l);
                if (!isfinite(f)) flags |= TT_FLAG_NONFINITE;
#pragma unroll
                for (int i = 0; i < K; ++i) acc[i] = fma(f, lam[i], acc[i]);
                busy = false;
            }
        }
        if constexpr (DEFER) {
            // deferred snaps (outside points; rare): one warp-cooperative nearest-element
            // search per pending lane, in lane order, then the owner adds f * lambda_j
            unsigned pm = __ballot_sync(FULL, pend_j >= 0);
            while (pm) {
                const int sl = __ffs(pm) - 1;
                pm &= pm - 1;
                double xe[D] = {};
                double lj[K];
                if (lane == sl) {
                    plan_lambda<D, PLAN>(plan, t.gid, e, pend_j, lj);
                    double vv[K][D];
                    vertices(vv);
                    map_point<D>(lj, vv, xe);
                }
#pragma unroll
                for (int c = 0; c < D; ++c) xe[c] = __shfl_sync(FULL, xe[c], sl);
                const int es = nearest_element_warp<D>(g, xe[0], xe[1], D == 3 ? xe[D - 1] : 0.0);
                if (lane == sl) {
                    double ls[K];
                    snap_lambda<D>(g, es, xe, ls);
                    const double f = (contrib || b) ? p1_eval<D>(src, es, ls) : 0.0;
                    if (!isfinite(f)) flags |= TT_FLAG_NONFINITE;
#pragma unroll
                    for (int i = 0; i < K; ++i) acc[i] = fma(f, lj[i], acc[i]);
                    pend_j = -1;
                }
            }
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1)
#pragma unroll
            for (int i = 0; i < K; ++i) acc[i] += __shfl_xor_sync(FULL, acc[i], off);
        if (active && sub_lane == 0) {
            const double q = (double)N * (1.0 / __ldg(t.measure + e));
            if (contrib) {
#pragma unroll
                for (int i = 0; i < K; ++i) contrib[cld ? i * cld + le : le * K + i] = acc[i] / q;
            } else if (b) {
#pragma unroll
                for (int i = 0; i < K; ++i) atomicAdd(b + __ldg(t.elems + e * K + i), acc[i] / q);
            }
        }
    }
    if (flags && status) atomicOr(status, flags);
}

template <int D>
__global__ void map_points_kernel(TargetDev t, int64_t e_lo, int64_t n_el, int plan_kind,
                                  PlanDev plan, double* __restrict__ pts) {
    constexpr int K = D + 1;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_el * plan.n) return;
    int64_t le = i / plan.n, j = i % plan.n, e = e_lo + le;
    double v[K][D];
    load_elem<D>(t, e, v);
    double lam[K];
    if (plan_kind == TT_PLAN_SHARED) {
        for (int c = 0; c < K; ++c) lam[c] = plan.lam[j * K + c];
    } else {
        philox_lambda<D>(plan.seed, stream_id(t.gid, e), j, lam);
    }
    double x[D];
    map_point<D>(lam, v, x);
    for (int c = 0; c < D; ++c) pts[i * D + c] = x[c];
}

template <int D, int SRC>
__global__ void eval_points_kernel(SrcDev src, const __grid_constant__ tt_expr_t expr,
                                   const double* __restrict__ pts, int64_t count,
                                   double* __restrict__ out, int32_t* __restrict__ status) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int flags = 0;
    if (i < count) {
        double x[D];
        for (int c = 0; c < D; ++c) x[c] = pts[i * D + c];
        int guess = -1;
        double f = eval_source<D, SRC>(src, expr, x, i, flags, guess);
        if (!isfinite(f)) flags |= TT_FLAG_NONFINITE;
        out[i] = f;
    }
    if (flags) atomicOr(status, flags);
}

__global__ void pack_coeffs_kernel(int64_t E, int k, const int32_t* __restrict__ elems,
                                   const double* __restrict__ coeffs, double* __restrict__ out) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < k; ++i) c[i] = coeffs[elems[e * k + i]];
    double2* o = reinterpret_cast<double2*>(out + e * 4);
    o[0] = make_double2(c[0], c[1]);
    o[1] = make_double2(c[2], c[3]);
}

// Per-element (gradient g, value at the origin vertex) of the P1 field: f = c_last +
// g.(x - v_last) on the element.  g solves E g = d with rows e_i = v_i - v_last and
// d_i = c_i - c_last (the walk record's binv is E^-T), via cross products / Cramer's rule
// from the vertex coordinates: the coordinates and coefficients are L2-resident gathers,
// so the kernel streams only the connectivity in and the 32 B records out.
template <int D>
__global__ void pack_grad_kernel(int64_t E, const int32_t* __restrict__ elems,
                                 const double* __restrict__ nodes, const double* __restrict__ coeffs,
                                 double* __restrict__ out) {
    constexpr int K = D + 1;
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    int n[K];
#pragma unroll
    for (int i = 0; i < K; ++i) n[i] = __ldg(elems + e * K + i);
    double v[K][D], c[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        c[i] = __ldg(coeffs + n[i]);
#pragma unroll
        for (int k = 0; k < D; ++k) v[i][k] = __ldg(nodes + (int64_t)n[i] * D + k);
    }
    double o[4] = {0.0, 0.0, 0.0, 0.0};
    o[D] = c[D];  // record = (g_0 .. g_{D-1}, c_last[, 0])
    if constexpr (D == 2) {
        const double a0 = v[0][0] - v[2][0], a1 = v[0][1] - v[2][1];
        const double b0 = v[1][0] - v[2][0], b1 = v[1][1] - v[2][1];
        const double d0 = c[0] - c[2], d1 = c[1] - c[2];
        const double inv = 1.0 / (a0 * b1 - a1 * b0);
        o[0] = (b1 * d0 - a1 * d1) * inv;
        o[1] = (a0 * d1 - b0 * d0) * inv;
    } else {
        double ed[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) ed[i][k] = v[i][k] - v[3][k];
        const auto cross = [](const double* x, const double* y, double* z) {
            z[0] = x[1] * y[2] - x[2] * y[1];
            z[1] = x[2] * y[0] - x[0] * y[2];
            z[2] = x[0] * y[1] - x[1] * y[0];
        };
        double c12[3], c20[3], c01[3];
        cross(ed[1], ed[2], c12);
        cross(ed[2], ed[0], c20);
        cross(ed[0], ed[1], c01);
        const double inv = 1.0 / (ed[0][0] * c12[0] + ed[0][1] * c12[1] + ed[0][2] * c12[2]);
        const double d0 = c[0] - c[3], d1 = c[1] - c[3], d2 = c[2] - c[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) o[k] = (d0 * c12[k] + d1 * c20[k] + d2 * c01[k]) * inv;
    }
    double2* q = reinterpret_cast<double2*>(out + e * 4);
    q[0] = make_double2(o[0], o[1]);
    q[1] = make_double2(o[2], o[3]);
}

// b[n] = sum over the node's incidences (e*k + a ascending) of contrib[e - e_lo, a],
// starting from 0.0 -- exactly np.add.at's accumulation order (montecarlo.py:146).
// Entry q = e*k + a is in the element range iff e_lo*k <= q < e_hi*k.  Row-major contrib
// (LD = false) is then read at q - e_lo*k; the transposed layout (LD: contrib[a*ld + e - e_lo],
// what the fused kernel writes for the node gather) at a*ld + e - e_lo -- there the gathers of
// a warp's consecutive nodes, which take the same vertex slot of elements a few ids apart on
// structured meshes, share lines (0.41 lines per gather at C2 instead of 1.0).  Index loads are
// 16-byte aligned int4 chunks covering the node's incidence range (two chunks = 8 positions per
// trip, out-of-range ones masked): 2 LDG.128 instead of 8 LDG.32 per trip; then the trip's (up
// to 8) independent contribution gathers, then the adds in ascending order.
template <int K, bool LD>
__global__ void reduce_nodes_kernel(int64_t n_nodes, const int64_t* __restrict__ inc_start,
                                    const int32_t* __restrict__ inc, int64_t e_lo, int64_t e_hi,
                                    int64_t ld, const double* __restrict__ contrib, double* __restrict__ b) {
    int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= n_nodes) return;
    const int64_t lo_k = e_lo * K, hi_k = e_hi * K;
    double s = 0.0;
    const int64_t q0 = __ldg(inc_start + n), q1 = __ldg(inc_start + n + 1);
    for (int64_t c = q0 & ~int64_t(3); c < q1; c += 8) {
        const int4 u = __ldg(reinterpret_cast<const int4*>(inc + c));
        const int4 w = c + 4 < q1 ? __ldg(reinterpret_cast<const int4*>(inc + c + 4)) : make_int4(0, 0, 0, 0);
        const int ea[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
        int64_t src[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            src[t] = -1;
            if (c + t >= q0 && c + t < q1 && ea[t] >= lo_k && ea[t] < hi_k) {
                if constexpr (LD) {
                    const int e = ea[t] / K;            // constant divisor
                    src[t] = (int64_t)(ea[t] - e * K) * ld + (e - e_lo);
                } else {
                    src[t] = ea[t] - lo_k;
                }
            }
        }
        double v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) v[t] = src[t] >= 0 ? __ldg(contrib + src[t]) : 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t)
            if (src[t] >= 0) s = add(s, v[t]);
    }
    b[n] = s;
}

__global__ void incidence_count_kernel(int64_t nent, const int32_t* __restrict__ elems,
                                       unsigned long long* __restrict__ counts) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nent) return;
    atomicAdd(counts + elems[q], 1ull);
}

__global__ void incidence_fill_kernel(int64_t nent, const int32_t* __restrict__ elems,
                                      unsigned long long* __restrict__ cursor,
                                      int32_t* __restrict__ inc) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nent) return;
    unsigned long long pos = atomicAdd(cursor + elems[q], 1ull);
    inc[pos] = (int32_t)q;  // q = e*k + a
}

__global__ void segment_sort_kernel2(int64_t nseg, const int64_t* __restrict__ start,
                                     int32_t* __restrict__ vals) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    int64_t a = start[s], b = start[s + 1];
    if (b - a <= 64) {  // (node incidences: ~23 in 3-D) sorted in a thread-local buffer
        int32_t buf[64];
        const int n = (int)(b - a);
        for (int i = 0; i < n; ++i) buf[i] = vals[a + i];
        for (int i = 1; i < n; ++i) {
            const int32_t v = buf[i];
            int j = i - 1;
            while (j >= 0 && buf[j] > v) { buf[j + 1] = buf[j]; --j; }
            buf[j + 1] = v;
        }
        for (int i = 0; i < n; ++i) vals[a + i] = buf[i];
        return;
    }
    for (int64_t i = a + 1; i < b; ++i) {
        int32_t v = vals[i];
        int64_t j = i - 1;
        while (j >= a && vals[j] > v) { vals[j + 1] = vals[j]; --j; }
        vals[j + 1] = v;
    }
}

static SrcDev to_src(const tt_source_t& s) {
    SrcDev d;
    d.kind = s.kind;
    d.outside = s.outside;
    d.grid = to_dev(s.grid);
    d.src_elems = s.src_elems;
    d.coeffs = s.coeffs;
    d.values = s.values;
    d.cached = s.cached_ids;
    d.seeds = s.seeds;
    d.ecoef = s.elem_coeffs;
    d.egrad = s.elem_grad;
    d.density = nullptr;
    return d;
}

// Resident blocks per SM of a kernel at a block size, queried once per kernel instance
// (every caller passes the same kernel/block/dynamic-smem triple).
template <class Kernel>
static int blocks_per_sm(Kernel kernel, int block, size_t smem) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, block, smem);
    return per < 1 ? 1 : per;
}

// Lanes per element for the fused mesh kernel.  Measured on C2 (ms per load): N = 32 / 48
// G = 4 0.694 / 0.927 vs G = 2 0.744 / 1.053; N = 64 G = 4 best (G = 8 +5 %); N = 128
// G = 4 ~ G = 8; N = 256 G = 16 3.76 vs G = 8 3.87; N = 512 G = 16 6.94 vs G = 32 7.35;
// N = 1024 G = 16 13.41 vs 13.68.  Other sources: ~16 samples per lane.
static int lanes_per_element(int src_kind, int64_t N) {
    if (src_kind == TT_SRC_MESH) return N < 32 ? 2 : N < 128 ? 4 : N < 512 ? 8 : N < 2048 ? 16 : 32;
    const int64_t g = N / 16;
    return g < 8 ? 4 : g < 16 ? 8 : g < 32 ? 16 : 32;
}

// The fused mesh-backed load (and, with ids != NULL, the id sink of tt_mc_cache_ids: the
// same kernel instance, so cached ids are exactly the ids every load walks to).
template <int D, int PLAN, int G>
static int launch_mesh(const TargetDev& td, int64_t e_lo, int64_t e_hi, const PlanDev& pd,
                       const SrcDev& sd, bool defer, double* contrib, int64_t cld, double* b, int32_t* ids,
                       int32_t* status, cudaStream_t st) {
    constexpr int EPW = 32 / G;
    const int64_t tiles = (e_hi - e_lo + EPW - 1) / EPW;
    // one wave of blocks (the per-block seed-slot table is built once; measured 0.08 ms
    // better than 16 waves at C2, N = 64); 32-lane groups (N >= 512) keep 16 waves (+1 %)
    const int waves = G >= 32 ? 16 : 1;
    const bool slot = PLAN == TT_PLAN_SHARED && pd.n <= kSlotCap;
    if (!slot) {   // per-element plans: the nearest-anchor lookup tables (built once)
        const int rc = anchor_tables_ready(st);
        if (rc) return rc;
    }
    // the walk order (tt_plan_walk_order) applies to the slot-table kernels only
    PlanDev pw = pd;
    if (!slot || !pd.order || !pd.lam_walk) pw.order = nullptr;
    else pw.lam = pd.lam_walk;
    // dynamic shared memory = the seed-slot table (N bytes, SLOT kernels only): every byte
    // of shared memory is L1 the walk's records lose (+20 KB/block costs 0.056 ms at C2)
    const size_t smem = slot ? (size_t)((pd.n + 15) / 16 * 16) : 0;
    auto go = [&](auto kernel) {
        static const int per = blocks_per_sm(kernel, kMcBlock, 0);
        constexpr int kWarps = kMcBlock / 32;  // a warp works one tile at a time
        int64_t nb = (tiles + kWarps - 1) / kWarps;
        const int64_t cap = (int64_t)sm_count() * per * waves;
        nb = nb > cap ? cap : nb < 1 ? 1 : nb;
        kernel<<<(unsigned)nb, kMcBlock, smem, st>>>(td, e_lo, e_hi, pw, sd, contrib, cld, b, ids, status);
    };
    // DEFER costs registers (C2: 1.12 -> 1.22 ms), so only pairs known to snap run it
    if constexpr (PLAN == TT_PLAN_SHARED) {
        if (slot) {
            if (defer) go(mc_mesh_kernel<D, PLAN, G, true, true>);
            else go(mc_mesh_kernel<D, PLAN, G, true, false>);
            return launch_check("mc_mesh_kernel");
        }
    }
    if (defer) go(mc_mesh_kernel<D, PLAN, G, false, true>);
    else go(mc_mesh_kernel<D, PLAN, G, false, false>);
    return launch_check("mc_mesh_kernel");
}

template <int D, int PLAN, int SRC, int G>
static int launch_mc(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                     const tt_source_t* s, double* contrib, int64_t cld, double* b, int32_t* ids,
                     int32_t* status, cudaStream_t st) {
    TargetDev td{t->nodes, t->elems, t->measure, t->gid};
    PlanDev pd{p->n_samples, p->lam, p->seed, p->order, p->lam_walk};
    SrcDev sd = to_src(*s);
    if constexpr (SRC == TT_SRC_MESH) {
        return launch_mesh<D, PLAN, G>(td, e_lo, e_hi, pd, sd, (s->hints & TT_HINT_DEFER_SNAP) != 0,
                                       contrib, cld, b, ids, status, st);
    } else {
        constexpr int EPW = 32 / G;
        const int64_t tiles = (e_hi - e_lo + EPW - 1) / EPW;
        static const int per = blocks_per_sm(mc_load_kernel<D, PLAN, SRC, G>, 256, 0);
        int64_t blocks = (tiles + 7) / 8;
        const int64_t cap = (int64_t)sm_count() * per * 16;
        blocks = blocks > cap ? cap : blocks < 1 ? 1 : blocks;
        mc_load_kernel<D, PLAN, SRC, G><<<(unsigned)blocks, 256, 0, st>>>(td, e_lo, e_hi, pd, sd,
                                                                          s->expr, contrib, cld, b, status);
        return launch_check("mc_load_kernel");
    }
}

template <int D, int PLAN, int SRC>
static int dispatch_g(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                      const tt_source_t* s, double* contrib, int64_t cld, double* b, int32_t* ids,
                      int32_t* status, cudaStream_t st) {
    const int G = lanes_per_element(SRC, p->n_samples);
    if constexpr (SRC == TT_SRC_MESH)
        if (G == 2) return launch_mc<D, PLAN, SRC, 2>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
    if (G == 4) return launch_mc<D, PLAN, SRC, 4>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
    if (G == 8) return launch_mc<D, PLAN, SRC, 8>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
    if (G == 16) return launch_mc<D, PLAN, SRC, 16>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
    return launch_mc<D, PLAN, SRC, 32>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
}

template <int D, int PLAN>
static int dispatch_src(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                        const tt_source_t* s, double* contrib, int64_t cld, double* b, int32_t* ids,
                        int32_t* status, cudaStream_t st) {
    switch (s->kind) {
        case TT_SRC_EXPR: return dispatch_g<D, PLAN, TT_SRC_EXPR>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
        case TT_SRC_MESH: return dispatch_g<D, PLAN, TT_SRC_MESH>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
        case TT_SRC_VALUES: return dispatch_g<D, PLAN, TT_SRC_VALUES>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
        case TT_SRC_CACHED: return dispatch_g<D, PLAN, TT_SRC_CACHED>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
    }
    set_error("tt_mc_load: unknown source kind %d", s->kind);
    return TT_ERR_INVALID_PARAMETER;
}

template <int D>
static int dispatch_plan(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                         const tt_source_t* s, double* contrib, int64_t cld, double* b, int32_t* ids,
                         int32_t* status, cudaStream_t st) {
    if (p->kind == TT_PLAN_SHARED) return dispatch_src<D, TT_PLAN_SHARED>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
    if (p->kind == TT_PLAN_PHILOX) return dispatch_src<D, TT_PLAN_PHILOX>(t, e_lo, e_hi, p, s, contrib, cld, b, ids, status, st);
    set_error("tt_mc_load: unknown plan kind %d", p->kind);
    return TT_ERR_INVALID_PARAMETER;
}

static int check_source(const tt_source_t* s, int dim) {
    if (!s) { set_error("null source"); return TT_ERR_INVALID_PARAMETER; }
    if (s->dim != dim) {
        set_error("source dimension %d does not match target dimension %d", s->dim, dim);
        return TT_ERR_DIMENSION_MISMATCH;
    }
    if (s->kind == TT_SRC_EXPR) {
        if (s->expr.n_ops < 1 || s->expr.n_ops > TT_EXPR_MAX_OPS) {
            set_error("expression program length %d out of range", s->expr.n_ops);
            return TT_ERR_INVALID_PARAMETER;
        }
    } else if (s->kind == TT_SRC_MESH) {
        if (s->grid.dim != dim || !s->grid.cell_start || !s->grid.rec || !s->coeffs || !s->src_elems) {
            set_error("mesh-backed source: incomplete descriptor or dimension mismatch");
            return TT_ERR_DIMENSION_MISMATCH;
        }
    } else if (s->kind == TT_SRC_CACHED) {
        if (s->grid.dim != dim || !s->grid.rec || !s->coeffs || !s->src_elems || !s->cached_ids) {
            set_error("cached source: incomplete descriptor or dimension mismatch");
            return TT_ERR_DIMENSION_MISMATCH;
        }
    } else if (s->kind == TT_SRC_VALUES) {
        if (!s->values) { set_error("values source without values"); return TT_ERR_INVALID_PARAMETER; }
    } else {
        set_error("unknown source kind %d", s->kind);
        return TT_ERR_INVALID_PARAMETER;
    }
    return TT_OK;
}

}  // namespace tt

using namespace tt;

extern "C" int tt_mc_load_ld(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                             const tt_source_t* s, double* contrib, int64_t contrib_ld, double* b,
                             int32_t* status, void* stream) {
    if (!t || !p || (t->dim != 2 && t->dim != 3) || p->dim != t->dim) {
        set_error("tt_mc_load: target/plan dimension mismatch");
        return TT_ERR_DIMENSION_MISMATCH;
    }
    if (e_lo < 0 || e_hi > t->n_elems || e_lo > e_hi || p->n_samples < 1) {
        set_error("tt_mc_load: bad element range or sample count");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (p->kind == TT_PLAN_SHARED && !p->lam) {
        set_error("tt_mc_load: shared plan without lambda table");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (contrib_ld != 0 && contrib_ld < e_hi - e_lo) {
        set_error("tt_mc_load_ld: contrib_ld smaller than the element range");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (!contrib && !b) {
        set_error("tt_mc_load: need contrib or b output");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (s && s->kind == TT_SRC_MESH && s->grid.walk && s->grid.wrec && s->seeds && !s->elem_grad) {
        // the compact walk's certified hits evaluate f from the gradient records
        set_error("tt_mc_load: a walk source (seeds + grid.wrec) needs elem_grad (tt_pack_grad)");
        return TT_ERR_INVALID_PARAMETER;
    }
    int st = check_source(s, t->dim);
    if (st) return st;
    if (e_hi == e_lo) return TT_OK;
    if (t->dim == 2) return dispatch_plan<2>(t, e_lo, e_hi, p, s, contrib, contrib_ld, b, nullptr, status, as_stream(stream));
    return dispatch_plan<3>(t, e_lo, e_hi, p, s, contrib, contrib_ld, b, nullptr, status, as_stream(stream));
}

// One block: each sample's nearest walk anchor (the fused kernel's rule), then a stable
// counting sort of the sample indices by anchor.
template <int D>
__global__ void walk_order_kernel(int64_t n, const double* __restrict__ lam, int32_t* __restrict__ order,
                                  double* __restrict__ lam_walk) {
    constexpr int K = D + 1;
    __shared__ int8_t s_key[kSlotCap];
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        double l[K];
#pragma unroll
        for (int a = 0; a < K; ++a) l[a] = lam[j * K + a];
        s_key[j] = (int8_t)seed_slot_nearest<D>(l, seeds_used(n));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int start[kSeeds + 1] = {0};
        for (int64_t j = 0; j < n; ++j) ++start[s_key[j] + 1];
        for (int k = 0; k < kSeeds; ++k) start[k + 1] += start[k];
        for (int64_t j = 0; j < n; ++j) order[start[s_key[j]]++] = (int32_t)j;
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < n * K; q += blockDim.x) lam_walk[q] = lam[(int64_t)order[q / K] * K + q % K];
}

extern "C" int tt_plan_walk_order(int dim, int64_t n_samples, const double* lam, int32_t* order,
                                  double* lam_walk, void* stream) {
    if ((dim != 2 && dim != 3) || n_samples < 1 || n_samples > kSlotCap || !lam || !order || !lam_walk) {
        set_error("tt_plan_walk_order: dim 2/3, 1 <= n_samples <= %d, lam, order and lam_walk required", kSlotCap);
        return TT_ERR_INVALID_PARAMETER;
    }
    if (dim == 2) walk_order_kernel<2><<<1, 256, 0, as_stream(stream)>>>(n_samples, lam, order, lam_walk);
    else walk_order_kernel<3><<<1, 256, 0, as_stream(stream)>>>(n_samples, lam, order, lam_walk);
    return launch_check("walk_order_kernel");
}

extern "C" int tt_mc_load(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                          const tt_source_t* s, double* contrib, double* b, int32_t* status,
                          void* stream) {
    return tt_mc_load_ld(t, e_lo, e_hi, p, s, contrib, 0, b, status, stream);
}

// Importance-weighted load (montecarlo.py:165-176): the simple sample loop (mc_load_kernel)
// for every source kind, f / (N p_j) per sample with the caller's densities.
template <int D, int SRC, int G>
static int launch_density(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                          const tt_source_t* s, const double* density, double* contrib,
                          int32_t* status, cudaStream_t st) {
    TargetDev td{t->nodes, t->elems, t->measure, t->gid};
    PlanDev pd{p->n_samples, p->lam, p->seed, p->order, p->lam_walk};
    SrcDev sd = to_src(*s);
    sd.density = density;
    constexpr int EPW = 32 / G;
    const int64_t tiles = (e_hi - e_lo + EPW - 1) / EPW;
    static const int per = blocks_per_sm(mc_load_kernel<D, TT_PLAN_SHARED, SRC, G>, 256, 0);
    int64_t blocks = (tiles + 7) / 8;
    const int64_t cap = (int64_t)sm_count() * per * 16;
    blocks = blocks > cap ? cap : blocks < 1 ? 1 : blocks;
    mc_load_kernel<D, TT_PLAN_SHARED, SRC, G><<<(unsigned)blocks, 256, 0, st>>>(td, e_lo, e_hi, pd, sd, s->expr,
                                                                               contrib, 0, nullptr, status);
    return launch_check("mc_load_kernel (density)");
}

template <int D, int SRC>
static int density_g(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                     const tt_source_t* s, const double* density, double* contrib, int32_t* status,
                     cudaStream_t st) {
    const int G = lanes_per_element(TT_SRC_VALUES, p->n_samples);
    if (G <= 4) return launch_density<D, SRC, 4>(t, e_lo, e_hi, p, s, density, contrib, status, st);
    if (G == 8) return launch_density<D, SRC, 8>(t, e_lo, e_hi, p, s, density, contrib, status, st);
    if (G == 16) return launch_density<D, SRC, 16>(t, e_lo, e_hi, p, s, density, contrib, status, st);
    return launch_density<D, SRC, 32>(t, e_lo, e_hi, p, s, density, contrib, status, st);
}

template <int D>
static int density_src(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                       const tt_source_t* s, const double* density, double* contrib, int32_t* status,
                       cudaStream_t st) {
    switch (s->kind) {
        case TT_SRC_EXPR: return density_g<D, TT_SRC_EXPR>(t, e_lo, e_hi, p, s, density, contrib, status, st);
        case TT_SRC_MESH: return density_g<D, TT_SRC_MESH>(t, e_lo, e_hi, p, s, density, contrib, status, st);
        case TT_SRC_VALUES: return density_g<D, TT_SRC_VALUES>(t, e_lo, e_hi, p, s, density, contrib, status, st);
    }
    set_error("tt_mc_load_density: unsupported source kind %d", s->kind);
    return TT_ERR_INVALID_PARAMETER;
}

extern "C" int tt_mc_load_density(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                                  const tt_source_t* s, const double* density, double* contrib,
                                  int32_t* status, void* stream) {
    if (!t || !p || (t->dim != 2 && t->dim != 3) || p->dim != t->dim || p->kind != TT_PLAN_SHARED || !p->lam) {
        set_error("tt_mc_load_density: needs a shared plan of the target's dimension");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (e_lo < 0 || e_hi > t->n_elems || e_lo > e_hi || p->n_samples < 1 || !density || !contrib) {
        set_error("tt_mc_load_density: bad element range, sample count or buffers");
        return TT_ERR_INVALID_PARAMETER;
    }
    int st = check_source(s, t->dim);
    if (st) return st;
    if (e_hi == e_lo) return TT_OK;
    if (t->dim == 2) return density_src<2>(t, e_lo, e_hi, p, s, density, contrib, status, as_stream(stream));
    return density_src<3>(t, e_lo, e_hi, p, s, density, contrib, status, as_stream(stream));
}

extern "C" int tt_mc_cache_ids(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                               const tt_grid_t* g, const int32_t* seeds, int32_t* ids, void* stream) {
    if (!t || !p || !g || p->dim != t->dim || g->dim != t->dim || e_lo < 0 || e_hi > t->n_elems ||
        e_lo > e_hi || !ids || (p->kind == TT_PLAN_SHARED && !p->lam)) {
        set_error("tt_mc_cache_ids: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    if ((e_hi - e_lo) * p->n_samples == 0) return TT_OK;
    // the fused load kernel itself (same instance the load launches for this N) with an id
    // sink and no accumulation, so cached ids are the ids every load sees (transfer.py:74-82)
    tt_source_t s{};
    s.kind = TT_SRC_MESH;
    s.outside = TT_OUTSIDE_SNAP;
    s.dim = t->dim;
    s.grid = *g;
    s.seeds = seeds;
    if (t->dim == 2) return dispatch_plan<2>(t, e_lo, e_hi, p, &s, nullptr, 0, nullptr, ids, nullptr, as_stream(stream));
    return dispatch_plan<3>(t, e_lo, e_hi, p, &s, nullptr, 0, nullptr, ids, nullptr, as_stream(stream));
}

extern "C" int tt_map_points(const tt_mesh_t* t, int64_t e_lo, int64_t e_hi, const tt_plan_t* p,
                             double* pts, void* stream) {
    if (!t || !p || p->dim != t->dim || e_lo < 0 || e_hi > t->n_elems || e_lo > e_hi) {
        set_error("tt_map_points: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    int64_t total = (e_hi - e_lo) * p->n_samples;
    if (total == 0) return TT_OK;
    TargetDev td{t->nodes, t->elems, t->measure, t->gid};
    PlanDev pd{p->n_samples, p->lam, p->seed, p->order, p->lam_walk};
    auto s = as_stream(stream);
    if (t->dim == 2)
        map_points_kernel<2><<<grid_for(total, 256), 256, 0, s>>>(td, e_lo, e_hi - e_lo, p->kind, pd, pts);
    else
        map_points_kernel<3><<<grid_for(total, 256), 256, 0, s>>>(td, e_lo, e_hi - e_lo, p->kind, pd, pts);
    return launch_check("map_points_kernel");
}

extern "C" int tt_eval_points(const tt_source_t* src, const double* pts, int64_t count,
                              double* out, int32_t* status, void* stream) {
    if (!src) { set_error("null source"); return TT_ERR_INVALID_PARAMETER; }
    const int dim = src->dim;
    if (dim != 2 && dim != 3) { set_error("tt_eval_points: source dim must be 2 or 3"); return TT_ERR_INVALID_PARAMETER; }
    int st = check_source(src, dim);
    if (st) return st;
    if (count == 0) return TT_OK;
    SrcDev sd = to_src(*src);
    auto s = as_stream(stream);
    const unsigned g = grid_for(count, 256);
    if (dim == 2) {
        if (src->kind == TT_SRC_EXPR) eval_points_kernel<2, TT_SRC_EXPR><<<g, 256, 0, s>>>(sd, src->expr, pts, count, out, status);
        else if (src->kind == TT_SRC_MESH) eval_points_kernel<2, TT_SRC_MESH><<<g, 256, 0, s>>>(sd, src->expr, pts, count, out, status);
        else eval_points_kernel<2, TT_SRC_VALUES><<<g, 256, 0, s>>>(sd, src->expr, pts, count, out, status);
    } else {
        if (src->kind == TT_SRC_EXPR) eval_points_kernel<3, TT_SRC_EXPR><<<g, 256, 0, s>>>(sd, src->expr, pts, count, out, status);
        else if (src->kind == TT_SRC_MESH) eval_points_kernel<3, TT_SRC_MESH><<<g, 256, 0, s>>>(sd, src->expr, pts, count, out, status);
        else eval_points_kernel<3, TT_SRC_VALUES><<<g, 256, 0, s>>>(sd, src->expr, pts, count, out, status);
    }
    return launch_check("eval_points_kernel");
}

extern "C" int tt_incidence_count(const tt_mesh_t* m, int64_t* inc_start, void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3)) {
        set_error("tt_incidence_count: bad mesh");
        return TT_ERR_INVALID_PARAMETER;
    }
    auto s = as_stream(stream);
    const int64_t nent = m->n_elems * (m->dim + 1);
    unsigned long long* counts = nullptr;
    int st = cuda_status(cudaMallocAsync((void**)&counts, sizeof(unsigned long long) * (m->n_nodes + 1), s),
                         "incidence counts alloc");
    if (st) return st;
    cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * (m->n_nodes + 1), s);
    cudaMemsetAsync(inc_start, 0, sizeof(int64_t), s);
    if (nent) incidence_count_kernel<<<grid_for(nent, 256), 256, 0, s>>>(nent, m->elems, counts);
    size_t tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, counts,
                                  reinterpret_cast<unsigned long long*>(inc_start + 1), m->n_nodes, s);
    void* tmp = nullptr;
    st = cuda_status(cudaMallocAsync(&tmp, tmp_bytes, s), "scan tmp alloc");
    if (!st) {
        cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, counts,
                                      reinterpret_cast<unsigned long long*>(inc_start + 1), m->n_nodes, s);
        st = launch_check("incidence count/scan");
        cudaFreeAsync(tmp, s);
    }
    cudaFreeAsync(counts, s);
    return st;
}

extern "C" int tt_incidence_fill(const tt_mesh_t* m, const int64_t* inc_start, int32_t* inc,
                                 int64_t* cursor, void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3)) {
        set_error("tt_incidence_fill: bad mesh");
        return TT_ERR_INVALID_PARAMETER;
    }
    const int64_t nent = m->n_elems * (m->dim + 1);
    if (nent >= 0x7fffffffLL) {
        set_error("tt_incidence_fill: e*k index exceeds int32");
        return TT_ERR_CAPACITY;
    }
    auto s = as_stream(stream);
    cudaMemcpyAsync(cursor, inc_start, sizeof(int64_t) * m->n_nodes, cudaMemcpyDeviceToDevice, s);
    if (nent)
        incidence_fill_kernel<<<grid_for(nent, 256), 256, 0, s>>>(
            nent, m->elems, reinterpret_cast<unsigned long long*>(cursor), inc);
    segment_sort_kernel2<<<grid_for(m->n_nodes, 256), 256, 0, s>>>(m->n_nodes, inc_start, inc);
    return launch_check("incidence fill/sort");
}

extern "C" int tt_reduce_nodes_ld(int64_t n_nodes, int k, const int64_t* inc_start, const int32_t* inc,
                                  int64_t e_lo, int64_t e_hi, const double* contrib, int64_t contrib_ld,
                                  double* b, void* stream) {
    if (n_nodes == 0) return TT_OK;
    if ((k != 1 && k != 3 && k != 4) || e_lo < 0 || contrib_ld < 0 || (k == 1 && contrib_ld)) {
        set_error("tt_reduce_nodes: k must be 1 (row-major only), 3 or 4; e_lo and contrib_ld >= 0");
        return TT_ERR_INVALID_PARAMETER;
    }
    // the int4 index loads read whole 16-byte chunks around a node's range (up to 3 entries
    // past the last one): inc must be 16-byte aligned and readable to a multiple of 4 entries
    if ((reinterpret_cast<uintptr_t>(inc) & 15) != 0) {
        set_error("tt_reduce_nodes: inc must be 16-byte aligned");
        return TT_ERR_INVALID_PARAMETER;
    }
    const int64_t hi = e_hi > (int64_t)INT32_MAX ? (int64_t)INT32_MAX : e_hi;   // entries are int32
    auto s = as_stream(stream);
    const unsigned grid = grid_for(n_nodes, 256);
    if (k == 1) {
        reduce_nodes_kernel<1, false><<<grid, 256, 0, s>>>(n_nodes, inc_start, inc, e_lo, hi, 0, contrib, b);
    } else if (k == 3) {
        if (contrib_ld) reduce_nodes_kernel<3, true><<<grid, 256, 0, s>>>(n_nodes, inc_start, inc, e_lo, hi, contrib_ld, contrib, b);
        else reduce_nodes_kernel<3, false><<<grid, 256, 0, s>>>(n_nodes, inc_start, inc, e_lo, hi, 0, contrib, b);
    } else {
        if (contrib_ld) reduce_nodes_kernel<4, true><<<grid, 256, 0, s>>>(n_nodes, inc_start, inc, e_lo, hi, contrib_ld, contrib, b);
        else reduce_nodes_kernel<4, false><<<grid, 256, 0, s>>>(n_nodes, inc_start, inc, e_lo, hi, 0, contrib, b);
    }
    return launch_check("reduce_nodes_kernel");
}

extern "C" int tt_reduce_nodes(int64_t n_nodes, int k, const int64_t* inc_start, const int32_t* inc,
                               int64_t e_lo, int64_t e_hi, const double* contrib, double* b,
                               void* stream) {
    return tt_reduce_nodes_ld(n_nodes, k, inc_start, inc, e_lo, e_hi, contrib, 0, b, stream);
}

extern "C" int tt_pack_coeffs(const tt_mesh_t* m, const double* coeffs, double* out, void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3) || !coeffs || !out) {
        set_error("tt_pack_coeffs: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (m->n_elems == 0) return TT_OK;
    pack_coeffs_kernel<<<grid_for(m->n_elems, 256), 256, 0, as_stream(stream)>>>(
        m->n_elems, m->dim + 1, m->elems, coeffs, out);
    return launch_check("pack_coeffs_kernel");
}

extern "C" int tt_pack_grad(const tt_mesh_t* m, const double* coeffs, double* out, void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3) || !m->nodes || !m->elems || !coeffs || !out) {
        set_error("tt_pack_grad: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (m->n_elems == 0) return TT_OK;
    if (m->dim == 2)
        pack_grad_kernel<2><<<grid_for(m->n_elems, 256), 256, 0, as_stream(stream)>>>(m->n_elems, m->elems, m->nodes, coeffs, out);
    else
        pack_grad_kernel<3><<<grid_for(m->n_elems, 256), 256, 0, as_stream(stream)>>>(m->n_elems, m->elems, m->nodes, coeffs, out);
    return launch_check("pack_grad_kernel");
}

#ifdef TT_MC_STATS
extern "C" int tt_debug_mc_stats(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_mc_stats, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_mc_stats, z, sizeof z);
    }
    return 0;
}
#endif
