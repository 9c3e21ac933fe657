// Shared device helpers for libtt_b200 (sm_100a).
//
// Bit-exactness contract: every operation that feeds an element id, a grid cell or a
// barycentric coordinate that the reference computes in plain IEEE double (numpy /
// Cython compiled without FMA, SURVEY.md finding 5) is written with the explicit
// round-to-nearest intrinsics below, which nvcc never contracts into DFMA.  Reductions
// whose order differs from the reference anyway (load vector sums, CG dots) may use FMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
#include "../../include/tt_b200.h"

#define TT_HD __host__ __device__ __forceinline__
#define TT_D __device__ __forceinline__

namespace tt {

// -------------------------------------------------------------- exact arithmetic
TT_D double mul(double a, double b) { return __dmul_rn(a, b); }
TT_D double add(double a, double b) { return __dadd_rn(a, b); }
TT_D double sub(double a, double b) { return __dsub_rn(a, b); }
TT_D double div(double a, double b) { return __ddiv_rn(a, b); }

// C `(int)t` as compiled for x86-64 (cvttsd2si): truncation, and INT_MIN for NaN or
// out-of-range values (the reference's `<int>` cast, _compiled.pyx:151-152).
TT_D int c_int_cast(double t) {
    return (t > -2147483649.0 && t < 2147483648.0) ? (int)t : (int)0x80000000;
}

// cell index along one axis: trunc(((v - lo) / (hi - lo)) * n), clamped to [0, n-1]
TT_D int axis_cell(double v, double lo, double hi, int n) {
    int i = c_int_cast(mul(div(sub(v, lo), sub(hi, lo)), (double)n));
    i = i < 0 ? 0 : i;
    return i > n - 1 ? n - 1 : i;
}

// -------------------------------------------------------------- error plumbing
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int launch_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    return cuda_status(e, what);
}

inline unsigned grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 0x7fffffff) g = 0x7fffffff;
    return (unsigned)g;
}

int sm_count();

// --------------------------------------------------------------- locate records
template <int D>
struct Rec {
    double b[D][D];
    double o[D];
};

// Packed record load: 2-D = 6 doubles of an 8-double (64 B) slot, 3-D = 12 of 16 (128 B).
template <int D>
TT_D void load_rec(const double* __restrict__ rec, int64_t e, Rec<D>& r) {
    if constexpr (D == 2) {
        const double2* p = reinterpret_cast<const double2*>(rec + e * 8);
        double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
        r.b[0][0] = a.x; r.b[0][1] = a.y; r.b[1][0] = b.x; r.b[1][1] = b.y;
        r.o[0] = c.x; r.o[1] = c.y;
    } else {
        const double2* p = reinterpret_cast<const double2*>(rec + e * 16);
        double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
        double2 d = __ldg(p + 3), f = __ldg(p + 4), g = __ldg(p + 5);
        r.b[0][0] = a.x; r.b[0][1] = a.y; r.b[0][2] = b.x;
        r.b[1][0] = b.y; r.b[1][1] = c.x; r.b[1][2] = c.y;
        r.b[2][0] = d.x; r.b[2][1] = d.y; r.b[2][2] = f.x;
        r.o[0] = f.y; r.o[1] = g.x; r.o[2] = g.y;
    }
}

// lambda_i = (b_i0*rx + b_i1*ry) [+ b_i2*rz]; lambda_last = ((1 - l0) - l1) [- l2]
// (_compiled.pyx:162-167; mesh.py:161-169)
template <int D>
TT_D void bary_from_rec(const Rec<D>& r, const double* x, double* lam) {
    double rel[D];
#pragma unroll
    for (int c = 0; c < D; ++c) rel[c] = sub(x[c], r.o[c]);
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double acc = add(mul(r.b[i][0], rel[0]), mul(r.b[i][1], rel[1]));
        if constexpr (D == 3) acc = add(acc, mul(r.b[i][2], rel[2]));
        lam[i] = acc;
    }
    double last = sub(sub(1.0, lam[0]), lam[1]);
    if constexpr (D == 3) last = sub(last, lam[2]);
    lam[D] = last;
}

template <int D>
TT_D bool inside_eps(const double* lam, double eps) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i <= D; ++i) ok = ok && (lam[i] >= -eps);
    return ok;
}

// point = ((l0*v0 + l1*v1) + l2*v2) [+ l3*v3] per coordinate (montecarlo.py:123-124)
template <int D>
TT_D void map_point(const double* lam, const double (*v)[D], double* x) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
        double acc = add(mul(lam[0], v[0][c]), mul(lam[1], v[1][c]));
        acc = add(acc, mul(lam[2], v[2][c]));
        if constexpr (D == 3) acc = add(acc, mul(lam[3], v[3][c]));
        x[c] = acc;
    }
}

// FMA point map for the certified walk: within 2 ulps of map_point; a certified element
// contains both points with a margin (>= 1e-12) far above that difference, so the id is
// the reference's; exact-scan fallbacks recompute x with map_point.
template <int D>
TT_D void map_point_fma(const double* lam, const double (*v)[D], double* x) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
        double acc = lam[0] * v[0][c];
        acc = fma(lam[1], v[1][c], acc);
        acc = fma(lam[2], v[2][c], acc);
        if constexpr (D == 3) acc = fma(lam[3], v[3][c], acc);
        x[c] = acc;
    }
}

// Record tail: certification margin and facet neighbours (written by walk prep).
template <int D>
struct RecTail {
    float tau;
    int nbr[D + 1];
};

template <int D>
TT_D void load_tail(const double* __restrict__ rec, int64_t e, RecTail<D>& t) {
    constexpr int S = (D == 2) ? 8 : 16;
    const int4* q = reinterpret_cast<const int4*>(rec + e * S + D * D + D);
    int4 a = __ldg(q);
    t.tau = __int_as_float(a.x);
    t.nbr[0] = a.y; t.nbr[1] = a.z; t.nbr[2] = a.w;
    if constexpr (D == 3) t.nbr[3] = __ldg(reinterpret_cast<const int*>(q + 1));
}

// Compact walk record: origin (double), binv (float), tau_f (float), nbr (int32).
template <int D>
struct WRec {
    double o[D];
    float b[D][D];
    float tau;
    int nbr[D + 1];
};

template <int D>
TT_D void load_wrec(const double* __restrict__ wrec, int64_t e, WRec<D>& w) {
    if constexpr (D == 2) {
        const int4* q = reinterpret_cast<const int4*>(wrec + e * 6);
        const int4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
        w.o[0] = __hiloint2double(a.y, a.x); w.o[1] = __hiloint2double(a.w, a.z);
        w.b[0][0] = __int_as_float(b.x); w.b[0][1] = __int_as_float(b.y);
        w.b[1][0] = __int_as_float(b.z); w.b[1][1] = __int_as_float(b.w);
        w.tau = __int_as_float(c.x);
        w.nbr[0] = c.y; w.nbr[1] = c.z; w.nbr[2] = c.w;
    } else {
        const int4* q = reinterpret_cast<const int4*>(wrec + e * 10);
        const int4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3), f = __ldg(q + 4);
        w.o[0] = __hiloint2double(a.y, a.x); w.o[1] = __hiloint2double(a.w, a.z);
        w.o[2] = __hiloint2double(b.y, b.x);
        w.b[0][0] = __int_as_float(b.z); w.b[0][1] = __int_as_float(b.w);
        w.b[0][2] = __int_as_float(c.x); w.b[1][0] = __int_as_float(c.y);
        w.b[1][1] = __int_as_float(c.z); w.b[1][2] = __int_as_float(c.w);
        w.b[2][0] = __int_as_float(d.x); w.b[2][1] = __int_as_float(d.y);
        w.b[2][2] = __int_as_float(d.z); w.tau = __int_as_float(d.w);
        w.nbr[0] = f.x; w.nbr[1] = f.y; w.nbr[2] = f.z; w.nbr[3] = f.w;
    }
}

// --------------------------------------------------------------- grid descriptor
struct GridDev {
    int n0, n1, n2;
    int walk;
    double lo[3], hi[3];
    const int64_t* __restrict__ cell_start;
    const int32_t* __restrict__ cell_elems;
    const double* __restrict__ rec;
    const double* __restrict__ centroids;
    const double* __restrict__ wrec;
};

inline GridDev to_dev(const tt_grid_t& g) {
    GridDev d;
    d.n0 = g.n[0]; d.n1 = g.n[1]; d.n2 = g.dim == 3 ? g.n[2] : 1;
    d.walk = g.walk;
    for (int c = 0; c < 3; ++c) { d.lo[c] = g.lo[c]; d.hi[c] = g.hi[c]; }
    d.cell_start = g.cell_start; d.cell_elems = g.cell_elems;
    d.rec = g.rec; d.centroids = g.centroids;
    d.wrec = g.wrec;
    return d;
}

template <int D>
TT_D int64_t point_cell(const GridDev& g, const double* x) {
    int ix = axis_cell(x[0], g.lo[0], g.hi[0], g.n0);
    int iy = axis_cell(x[1], g.lo[1], g.hi[1], g.n1);
    int64_t c = (int64_t)ix * g.n1 + iy;
    if constexpr (D == 3) c = c * g.n2 + axis_cell(x[2], g.lo[2], g.hi[2], g.n2);
    return c;
}

// First ascending candidate of the point's cell whose lambdas are all >= -eps
// (_compiled.pyx:147-174).  Returns -1 (OUTSIDE) when none qualifies.
template <int D>
TT_D int locate_point(const GridDev& g, const double* x, double eps, double* lam) {
    int64_t c = point_cell<D>(g, x);
    int64_t j0 = __ldg(g.cell_start + c), j1 = __ldg(g.cell_start + c + 1);
    for (int64_t j = j0; j < j1; ++j) {
        int e = __ldg(g.cell_elems + j);
        Rec<D> r;
        load_rec<D>(g.rec, e, r);
        double l[D + 1];
        bary_from_rec<D>(r, x, l);
        if (inside_eps<D>(l, eps)) {
#pragma unroll
            for (int i = 0; i <= D; ++i) lam[i] = l[i];
            return e;
        }
    }
    return -1;
}

// Certified facet walk.  From `guess`, evaluate lambda in the current element A (the
// reference formula, bit-identical); if min_i lambda_i >= tau_A the point lies at
// distance > k*eps*diam_max from every other element of a valid tessellation, so A is
// the ONLY element passing the reference predicate (lambda >= -eps) and therefore the
// element the reference's ascending cell scan returns (A is in the point's cell list
// because the cell map is monotone).  Otherwise step across the facet of the most
// negative lambda.  Anything uncertain (near a facet, boundary, step cap) falls back to
// the exact reference scan.  Returns the element or -1 (outside), lam filled as locate.
template <int D>
TT_D int locate_walk(const GridDev& g, const double* x, double eps, int guess, double* lam) {
    int e = guess;
#pragma unroll 1
    for (int step = 0; step < 12 && e >= 0; ++step) {
        Rec<D> r;
        load_rec<D>(g.rec, e, r);
        RecTail<D> t;
        load_tail<D>(g.rec, e, t);
        double l[D + 1];
        bary_from_rec<D>(r, x, l);
        int imin = 0;
        double lmin = l[0];
#pragma unroll
        for (int i = 1; i <= D; ++i)
            if (l[i] < lmin) { lmin = l[i]; imin = i; }
        if (lmin >= (double)t.tau) {
#pragma unroll
            for (int i = 0; i <= D; ++i) lam[i] = l[i];
            return e;
        }
        if (lmin >= -eps) break;  // inside within the slack but not certified: exact scan
        int nb = t.nbr[0];
#pragma unroll
        for (int i = 1; i <= D; ++i)
            if (imin == i) nb = t.nbr[i];
        e = nb;
    }
    return locate_point<D>(g, x, eps, lam);
}

// Expanding-ring nearest centroid, lowest id on ties, stop one ring after the first
// non-empty ring (locate.py:97-127).  d2 = (dx*dx + dy*dy) [+ dz*dz].
template <int D>
TT_D int nearest_element(const GridDev& g, const double* x) {
    int home[3];
    const int n[3] = {g.n0, g.n1, g.n2};
    for (int c = 0; c < D; ++c) {
        double t = mul(div(sub(x[c], g.lo[c]), sub(g.hi[c], g.lo[c])), (double)n[c]);
        // np.clip(t, 0, n-1) then int(): clip in double first (locate.py:102-103)
        t = t < 0.0 ? 0.0 : t;
        t = t > (double)(n[c] - 1) ? (double)(n[c] - 1) : t;
        home[c] = (int)t;
    }
    if constexpr (D == 2) home[2] = 0;
    int best = -1;
    double best_d2 = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    int first = -1;
    int max_ring = n[0] > n[1] ? n[0] : n[1];
    if constexpr (D == 3) max_ring = max_ring > n[2] ? max_ring : n[2];
    for (int ring = 0; ring <= max_ring; ++ring) {
        if (first >= 0 && ring > first + 1) break;
        const int rz = (D == 3) ? ring : 0;
        for (int cx = home[0] - ring; cx <= home[0] + ring; ++cx) {
            if (cx < 0 || cx >= n[0]) continue;
            for (int cy = home[1] - ring; cy <= home[1] + ring; ++cy) {
                if (cy < 0 || cy >= n[1]) continue;
                for (int cz = home[2] - rz; cz <= home[2] + rz; ++cz) {
                    if (cz < 0 || cz >= n[2]) continue;
                    int dx = abs(cx - home[0]), dy = abs(cy - home[1]), dz = abs(cz - home[2]);
                    int cheb = dx > dy ? dx : dy;
                    cheb = cheb > dz ? cheb : dz;
                    if (cheb != ring) continue;
                    int64_t c = ((int64_t)cx * n[1] + cy) * n[2] + cz;
                    int64_t j0 = g.cell_start[c], j1 = g.cell_start[c + 1];
                    for (int64_t j = j0; j < j1; ++j) {
                        int e = g.cell_elems[j];
                        double d2 = 0.0;
                        {
                            double d0 = sub(g.centroids[(int64_t)e * D + 0], x[0]);
                            double d1 = sub(g.centroids[(int64_t)e * D + 1], x[1]);
                            d2 = add(mul(d0, d0), mul(d1, d1));
                            if constexpr (D == 3) {
                                double dd = sub(g.centroids[(int64_t)e * D + 2], x[2]);
                                d2 = add(d2, mul(dd, dd));
                            }
                        }
                        if (d2 < best_d2 || (d2 == best_d2 && e < best)) { best = e; best_d2 = d2; }
                        if (first < 0) first = ring;
                    }
                }
            }
        }
    }
    return best;
}

// nearest_element with the 32 lanes of a warp cooperating (all lanes call it with the same
// x): each ring's cells are dealt out to the lanes, every lane keeps the lexicographic
// minimum of (d2, id) over its candidates, the ring bookkeeping (first non-empty ring, stop
// one ring later) is warp-uniform, and a shuffle tree takes the minimum over the lanes.
// The minimum of (d2, id) does not depend on the order candidates are visited, so the
// result is nearest_element's, bit for bit.
template <int D>
__device__ __noinline__ int nearest_element_warp(const GridDev g, double x0, double x1, double x2) {
    const double x[3] = {x0, x1, x2};
    const int lane = threadIdx.x & 31;
    int home[3];
    const int n[3] = {g.n0, g.n1, g.n2};
    for (int c = 0; c < D; ++c) {
        double t = mul(div(sub(x[c], g.lo[c]), sub(g.hi[c], g.lo[c])), (double)n[c]);
        t = t < 0.0 ? 0.0 : t;
        t = t > (double)(n[c] - 1) ? (double)(n[c] - 1) : t;
        home[c] = (int)t;
    }
    if constexpr (D == 2) home[2] = 0;
    int best = -1;
    double best_d2 = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    int first = -1;
    int max_ring = n[0] > n[1] ? n[0] : n[1];
    if constexpr (D == 3) max_ring = max_ring > n[2] ? max_ring : n[2];
    for (int ring = 0; ring <= max_ring; ++ring) {
        if (first >= 0 && ring > first + 1) break;
        const int side = 2 * ring + 1;
        const int rz = (D == 3) ? ring : 0;
        const int64_t cube = (int64_t)side * side * (D == 3 ? side : 1);
        bool found = false;
        for (int64_t q = lane; q < cube; q += 32) {
            const int cx = home[0] - ring + (int)(q % side);
            const int cy = home[1] - ring + (int)((q / side) % side);
            const int cz = home[2] - rz + (D == 3 ? (int)(q / ((int64_t)side * side)) : 0);
            if (cx < 0 || cx >= n[0] || cy < 0 || cy >= n[1] || cz < 0 || cz >= n[2]) continue;
            const int dx = abs(cx - home[0]), dy = abs(cy - home[1]), dz = abs(cz - home[2]);
            int cheb = dx > dy ? dx : dy;
            cheb = cheb > dz ? cheb : dz;
            if (cheb != ring) continue;
            const int64_t c = ((int64_t)cx * n[1] + cy) * n[2] + cz;
            const int64_t j0 = __ldg(g.cell_start + c), j1 = __ldg(g.cell_start + c + 1);
            for (int64_t j = j0; j < j1; ++j) {
                const int e = __ldg(g.cell_elems + j);
                const double d0 = sub(__ldg(g.centroids + (int64_t)e * D + 0), x[0]);
                const double d1 = sub(__ldg(g.centroids + (int64_t)e * D + 1), x[1]);
                double d2 = add(mul(d0, d0), mul(d1, d1));
                if constexpr (D == 3) {
                    const double dd = sub(__ldg(g.centroids + (int64_t)e * D + 2), x[2]);
                    d2 = add(d2, mul(dd, dd));
                }
                if (d2 < best_d2 || (d2 == best_d2 && e < best)) { best = e; best_d2 = d2; }
                found = true;
            }
        }
        if (first < 0 && __any_sync(0xffffffffu, found)) first = ring;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, best_d2, off);
        const int oe = __shfl_xor_sync(0xffffffffu, best, off);
        if (oe >= 0 && (best < 0 || od < best_d2 || (od == best_d2 && oe < best))) { best = oe; best_d2 = od; }
    }
    return best;
}

// Snapped barycentrics: clip(lambda, 0) / sum (montecarlo.py:58-63)
template <int D>
TT_D void snap_lambda(const GridDev& g, int e, const double* x, double* lam) {
    Rec<D> r;
    load_rec<D>(g.rec, e, r);
    bary_from_rec<D>(r, x, lam);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i <= D; ++i) {
        lam[i] = lam[i] < 0.0 ? 0.0 : lam[i];
    }
    s = add(lam[0], lam[1]);
#pragma unroll
    for (int i = 2; i <= D; ++i) s = add(s, lam[i]);
#pragma unroll
    for (int i = 0; i <= D; ++i) lam[i] = div(lam[i], s);
}

// Out-of-line snap for OUTSIDE points (rare): keeps the ring search's registers and
// stack out of the fused kernels' hot loops.
template <int D>
struct SnapOut {
    int e;
    double l[D + 1];
};

template <int D>
__device__ __noinline__ SnapOut<D> snap_point(const GridDev g, double x0, double x1, double x2) {
    const double x[3] = {x0, x1, x2};
    SnapOut<D> o;
    o.e = nearest_element<D>(g, x);
    snap_lambda<D>(g, o.e, x, o.l);
    return o;
}

// Walk-seed anchors in barycentric coordinates (scripts/seed_anchors.py): the first k+1
// are the centroid and the corner points (v_i + c)/2, the rest k-means centres of the
// uniform simplex with those fixed (anchors 16..47: k-means with the first 16 fixed).  A
// target element keeps the source element of each anchor (tt_seed_elements); a sample
// starts its walk at its nearest anchor's element, among the first seeds_used(N).
constexpr int kSeeds = TT_SEED_ANCHORS;
// anchors a plan of N samples per element walks from: the 16-anchor set below N = 32 (staging
// 48 seeds per element costs more than they save there), all 48 above
TT_D int seeds_used(int64_t n) { return n < 32 ? 16 : kSeeds; }
static __constant__ double kAnchor2[TT_SEED_ANCHORS][3] = {
    {0.333333, 0.333333, 0.333333},
    {0.666667, 0.166667, 0.166667},
    {0.166667, 0.666667, 0.166667},
    {0.166667, 0.166667, 0.666667},
    {0.363773, 0.564304, 0.071923},
    {0.106860, 0.449307, 0.443833},
    {0.085589, 0.834295, 0.080116},
    {0.070230, 0.624320, 0.305449},
    {0.531959, 0.357019, 0.111022},
    {0.532957, 0.113448, 0.353596},
    {0.083635, 0.082097, 0.834268},
    {0.367931, 0.073020, 0.559049},
    {0.069731, 0.308081, 0.622189},
    {0.268066, 0.246854, 0.485080},
    {0.274587, 0.482372, 0.243041},
    {0.832589, 0.083788, 0.083623},
    {0.169743, 0.254002, 0.576256},
    {0.056970, 0.783038, 0.159992},
    {0.452158, 0.314733, 0.233109},
    {0.434587, 0.224555, 0.340858},
    {0.264135, 0.570182, 0.165683},
    {0.040166, 0.916406, 0.043428},
    {0.471836, 0.055091, 0.473073},
    {0.173419, 0.344950, 0.481631},
    {0.181163, 0.764358, 0.054479},
    {0.557523, 0.182513, 0.259964},
    {0.765195, 0.179134, 0.055671},
    {0.465860, 0.476520, 0.057621},
    {0.389092, 0.431111, 0.179797},
    {0.669640, 0.273547, 0.056812},
    {0.282362, 0.052298, 0.665339},
    {0.270939, 0.155945, 0.573116},
    {0.053372, 0.241222, 0.705406},
    {0.586146, 0.037111, 0.376743},
    {0.050478, 0.706652, 0.242871},
    {0.163670, 0.537528, 0.298801},
    {0.040965, 0.041915, 0.917120},
    {0.574909, 0.258274, 0.166817},
    {0.227552, 0.406878, 0.365570},
    {0.046309, 0.541741, 0.411950},
    {0.582956, 0.380881, 0.036163},
    {0.056380, 0.162009, 0.781611},
    {0.764546, 0.054446, 0.181007},
    {0.046997, 0.414223, 0.538779},
    {0.277374, 0.668608, 0.054018},
    {0.378926, 0.173988, 0.447086},
    {0.666427, 0.061959, 0.271614},
    {0.183569, 0.053633, 0.762798},
};
static __constant__ double kAnchor3[TT_SEED_ANCHORS][4] = {
    {0.250000, 0.250000, 0.250000, 0.250000},
    {0.625000, 0.125000, 0.125000, 0.125000},
    {0.125000, 0.625000, 0.125000, 0.125000},
    {0.125000, 0.125000, 0.625000, 0.125000},
    {0.125000, 0.125000, 0.125000, 0.625000},
    {0.774629, 0.074457, 0.075479, 0.075435},
    {0.465274, 0.310278, 0.118290, 0.106158},
    {0.109478, 0.385985, 0.392791, 0.111746},
    {0.129884, 0.111950, 0.465907, 0.292258},
    {0.103289, 0.395581, 0.111945, 0.389184},
    {0.293299, 0.465529, 0.115429, 0.125743},
    {0.391758, 0.113144, 0.393580, 0.101518},
    {0.302490, 0.126738, 0.106420, 0.464352},
    {0.074152, 0.074355, 0.075047, 0.776447},
    {0.466578, 0.101469, 0.125798, 0.306155},
    {0.101515, 0.122250, 0.313852, 0.462382},
    {0.063933, 0.245468, 0.077921, 0.612679},
    {0.608135, 0.059137, 0.059237, 0.273491},
    {0.283735, 0.066270, 0.576581, 0.073414},
    {0.279410, 0.056537, 0.068463, 0.595590},
    {0.197913, 0.486010, 0.250019, 0.066059},
    {0.252762, 0.621449, 0.061466, 0.064322},
    {0.198399, 0.249127, 0.089889, 0.462585},
    {0.070729, 0.070262, 0.780078, 0.078930},
    {0.615924, 0.259115, 0.063440, 0.061521},
    {0.069649, 0.063014, 0.261468, 0.605869},
    {0.072629, 0.263610, 0.403667, 0.260094},
    {0.057433, 0.392253, 0.059064, 0.491249},
    {0.458579, 0.056868, 0.264019, 0.220534},
    {0.073220, 0.577189, 0.067393, 0.282198},
    {0.315215, 0.326331, 0.287626, 0.070827},
    {0.066681, 0.784638, 0.072828, 0.075853},
    {0.057414, 0.460041, 0.245565, 0.236980},
    {0.226274, 0.230979, 0.452730, 0.090017},
    {0.585864, 0.057747, 0.291082, 0.065306},
    {0.488256, 0.225142, 0.063454, 0.223148},
    {0.065619, 0.249334, 0.601710, 0.083337},
    {0.274382, 0.076993, 0.402860, 0.245766},
    {0.366722, 0.194431, 0.232084, 0.206763},
    {0.059898, 0.399546, 0.483900, 0.056657},
    {0.335557, 0.265694, 0.078096, 0.320653},
    {0.076038, 0.269712, 0.242520, 0.411730},
    {0.428332, 0.446604, 0.059943, 0.065122},
    {0.180265, 0.372359, 0.220818, 0.226558},
    {0.479605, 0.202734, 0.249930, 0.067731},
    {0.247756, 0.425914, 0.062073, 0.264257},
    {0.059260, 0.594713, 0.280503, 0.065524},
    {0.269916, 0.075857, 0.255810, 0.398417},
};

template <int D>
TT_D double anchor(int m, int a) { return D == 2 ? kAnchor2[m][a] : kAnchor3[m][a]; }

// Out-of-line exact localisation for the fused kernels' rare paths: the double-precision
// certified walk from `guess` (the element whose compact float test was inside its
// uncertainty band -- nearly always certified here in one step) and the reference cell scan
// when that is uncertain too, or directly the scan when guess < 0.  Out of line so the
// single diverged lane costs the hot loop no registers.
template <int D>
struct LocOut {
    int e;
    double l[D + 1];
};

template <int D>
__device__ __noinline__ LocOut<D> locate_from(const GridDev g, int guess, double x0, double x1, double x2,
                                              double eps) {
    const double x[3] = {x0, x1, x2};
    LocOut<D> o;
    o.e = guess >= 0 ? locate_walk<D>(g, x, eps, guess, o.l) : locate_point<D>(g, x, eps, o.l);
    return o;
}

}  // namespace tt
