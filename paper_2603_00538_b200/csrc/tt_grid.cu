// Mesh geometry and the uniform-grid point locator (locate.py:18-130, mesh.py:24-169).
//
// grid build: count (one atomic per (element, cell) pair) -> CUB inclusive scan ->
// atomic-cursor fill -> per-cell ascending sort.  The result is the reference's
// stable-argsort CSR (locate.py:65-70) exactly, independent of atomic ordering.
#include <cub/cub.cuh>
#include "tt_common.cuh"

namespace tt {

template <int D>
__global__ void geometry_kernel(int64_t E, const double* __restrict__ nodes,
                                const int32_t* __restrict__ elems, double* __restrict__ smeas,
                                double* __restrict__ rec, double* __restrict__ cent) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    constexpr int K = D + 1;
    double v[K][D];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        int64_t n = elems[e * K + i];
#pragma unroll
        for (int c = 0; c < D; ++c) v[i][c] = nodes[n * D + c];
    }
    if (smeas) {
        if constexpr (D == 2) {
            // 0.5 * ((b-a)x (c-a)y - (c-a)x (b-a)y)   mesh.py:24-29
            double t1 = mul(sub(v[1][0], v[0][0]), sub(v[2][1], v[0][1]));
            double t2 = mul(sub(v[2][0], v[0][0]), sub(v[1][1], v[0][1]));
            smeas[e] = mul(0.5, sub(t1, t2));
        } else {
            double u[3], w[3], t[3];
            for (int c = 0; c < 3; ++c) {
                u[c] = sub(v[1][c], v[0][c]);
                w[c] = sub(v[2][c], v[0][c]);
                t[c] = sub(v[3][c], v[0][c]);
            }
            double cx = sub(mul(w[1], t[2]), mul(w[2], t[1]));
            double cy = sub(mul(w[2], t[0]), mul(w[0], t[2]));
            double cz = sub(mul(w[0], t[1]), mul(w[1], t[0]));
            smeas[e] = div(add(add(mul(u[0], cx), mul(u[1], cy)), mul(u[2], cz)), 6.0);
        }
    }
    if (rec) {
        constexpr int S = (D == 2) ? 8 : 16;
        double* r = rec + e * S;
        if constexpr (D == 2) {
            // mesh.py:148-159
            double d0x = sub(v[0][0], v[2][0]), d0y = sub(v[0][1], v[2][1]);
            double d1x = sub(v[1][0], v[2][0]), d1y = sub(v[1][1], v[2][1]);
            double det = sub(mul(d0x, d1y), mul(d1x, d0y));
            r[0] = div(d1y, det);
            r[1] = div(-d1x, det);
            r[2] = div(-d0y, det);
            r[3] = div(d0x, det);
            r[4] = v[2][0];
            r[5] = v[2][1];
            r[6] = 0.0;
            r[7] = 0.0;
        } else {
            double a[3], b[3], c[3];
            for (int q = 0; q < 3; ++q) {
                a[q] = sub(v[0][q], v[3][q]);
                b[q] = sub(v[1][q], v[3][q]);
                c[q] = sub(v[2][q], v[3][q]);
            }
            double row[3][3];
            // rows: b x c, c x a, a x b
            row[0][0] = sub(mul(b[1], c[2]), mul(b[2], c[1]));
            row[0][1] = sub(mul(b[2], c[0]), mul(b[0], c[2]));
            row[0][2] = sub(mul(b[0], c[1]), mul(b[1], c[0]));
            row[1][0] = sub(mul(c[1], a[2]), mul(c[2], a[1]));
            row[1][1] = sub(mul(c[2], a[0]), mul(c[0], a[2]));
            row[1][2] = sub(mul(c[0], a[1]), mul(c[1], a[0]));
            row[2][0] = sub(mul(a[1], b[2]), mul(a[2], b[1]));
            row[2][1] = sub(mul(a[2], b[0]), mul(a[0], b[2]));
            row[2][2] = sub(mul(a[0], b[1]), mul(a[1], b[0]));
            double det = add(add(mul(a[0], row[0][0]), mul(a[1], row[0][1])), mul(a[2], row[0][2]));
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) r[i * 3 + j] = div(row[i][j], det);
            r[9] = v[3][0];
            r[10] = v[3][1];
            r[11] = v[3][2];
            r[12] = r[13] = r[14] = r[15] = 0.0;
        }
    }
    if (cent) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double s = add(v[0][c], v[1][c]);
#pragma unroll
            for (int i = 2; i < K; ++i) s = add(s, v[i][c]);
            cent[e * D + c] = div(s, (double)K);
        }
    }
}

__global__ void bbox_partial_kernel(int dim, int64_t n, const double* __restrict__ nodes,
                                    double* __restrict__ part) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        for (int c = 0; c < dim; ++c) {
            double v = nodes[i * dim + c];
            lo[c] = fmin(lo[c], v);
            hi[c] = fmax(hi[c], v);
        }
    }
    __shared__ double slo[3][256], shi[3][256];
    for (int c = 0; c < 3; ++c) { slo[c][threadIdx.x] = lo[c]; shi[c][threadIdx.x] = hi[c]; }
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int c = 0; c < 3; ++c) {
                slo[c][threadIdx.x] = fmin(slo[c][threadIdx.x], slo[c][threadIdx.x + s]);
                shi[c][threadIdx.x] = fmax(shi[c][threadIdx.x], shi[c][threadIdx.x + s]);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int c = 0; c < 3; ++c) {
            part[blockIdx.x * 6 + c] = slo[c][0];
            part[blockIdx.x * 6 + 3 + c] = shi[c][0];
        }
}

__global__ void bbox_final_kernel(int dim, int nparts, const double* __restrict__ part,
                                  double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int c = 0; c < dim; ++c) {
        double lo = INFINITY, hi = -INFINITY;
        for (int p = 0; p < nparts; ++p) {
            lo = fmin(lo, part[p * 6 + c]);
            hi = fmax(hi, part[p * 6 + 3 + c]);
        }
        out[c] = lo;
        out[dim + c] = hi;
    }
}

// per-element bbox cell range, cells of the reference binning (locate.py:42-53)
template <int D>
__device__ __forceinline__ void elem_cell_range(const GridDev& g, const double* __restrict__ nodes,
                                                const int32_t* __restrict__ elems, int64_t e,
                                                int lo_i[3], int hi_i[3]) {
    constexpr int K = D + 1;
    double mn[3], mx[3];
    for (int c = 0; c < D; ++c) { mn[c] = INFINITY; mx[c] = -INFINITY; }
    for (int i = 0; i < K; ++i) {
        int64_t n = elems[e * K + i];
        for (int c = 0; c < D; ++c) {
            double v = nodes[n * D + c];
            mn[c] = fmin(mn[c], v);
            mx[c] = fmax(mx[c], v);
        }
    }
    const int n[3] = {g.n0, g.n1, g.n2};
    for (int c = 0; c < D; ++c) {
        lo_i[c] = axis_cell(mn[c], g.lo[c], g.hi[c], n[c]);
        hi_i[c] = axis_cell(mx[c], g.lo[c], g.hi[c], n[c]);
    }
    if constexpr (D == 2) { lo_i[2] = 0; hi_i[2] = 0; }
}

template <int D>
__global__ void grid_count_kernel(GridDev g, int64_t E, const double* __restrict__ nodes,
                                  const int32_t* __restrict__ elems,
                                  unsigned long long* __restrict__ counts) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    int lo[3], hi[3];
    elem_cell_range<D>(g, nodes, elems, e, lo, hi);
    for (int ix = lo[0]; ix <= hi[0]; ++ix)
        for (int iy = lo[1]; iy <= hi[1]; ++iy)
            for (int iz = lo[2]; iz <= hi[2]; ++iz) {
                int64_t c = ((int64_t)ix * g.n1 + iy) * g.n2 + iz;
                atomicAdd(counts + c, 1ull);
            }
}

template <int D>
__global__ void grid_fill_kernel(GridDev g, int64_t E, const double* __restrict__ nodes,
                                 const int32_t* __restrict__ elems,
                                 unsigned long long* __restrict__ cursor,
                                 int32_t* __restrict__ cell_elems) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    int lo[3], hi[3];
    elem_cell_range<D>(g, nodes, elems, e, lo, hi);
    for (int ix = lo[0]; ix <= hi[0]; ++ix)
        for (int iy = lo[1]; iy <= hi[1]; ++iy)
            for (int iz = lo[2]; iz <= hi[2]; ++iz) {
                int64_t c = ((int64_t)ix * g.n1 + iy) * g.n2 + iz;
                unsigned long long pos = atomicAdd(cursor + c, 1ull);
                cell_elems[pos] = (int32_t)e;
            }
}

// ascending sort of each CSR segment (segments are short: ~6 (2-D) to ~25 (3-D) ids).  A
// segment of up to 64 ids is sorted in a thread-local buffer (L1-resident) instead of with
// dependent global-memory round trips; longer ones in place.
__global__ void segment_sort_kernel(int64_t nseg, const int64_t* __restrict__ start,
                                    int32_t* __restrict__ vals) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    const int64_t a = start[s], b = start[s + 1];
    if (b - a <= 64) {
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

template <int D>
__global__ void locate_kernel(GridDev g, const double* __restrict__ pts, int64_t K, double eps,
                              int32_t* __restrict__ elem, double* __restrict__ lam) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= K) return;
    double x[D], l[D + 1];
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = pts[i * D + c];
    int e = locate_point<D>(g, x, eps, l);
    elem[i] = e;
#pragma unroll
    for (int c = 0; c <= D; ++c) lam[i * (D + 1) + c] = (e >= 0) ? l[c] : 0.0;
}

// The reference seam's own argument layout: binv (E,2,2) and origin (E,2) as separate
// arrays (_compiled.pyx:127-175).
__global__ void locate_many_seam_kernel(const double* __restrict__ pts, int64_t K, int nx, int ny,
                                        double xmin, double ymin, double xmax, double ymax,
                                        const int64_t* __restrict__ cstart,
                                        const int32_t* __restrict__ celems,
                                        const double* __restrict__ binv,
                                        const double* __restrict__ origin, double eps,
                                        int32_t* __restrict__ elem, double* __restrict__ lam) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= K) return;
    double x[2] = {pts[2 * p], pts[2 * p + 1]};
    int ix = axis_cell(x[0], xmin, xmax, nx);
    int iy = axis_cell(x[1], ymin, ymax, ny);
    int64_t c = (int64_t)ix * ny + iy;
    int found = -1;
    double l[3] = {0.0, 0.0, 0.0};
    for (int64_t j = cstart[c]; j < cstart[c + 1]; ++j) {
        int e = celems[j];
        Rec<2> r;
        r.b[0][0] = binv[e * 4 + 0]; r.b[0][1] = binv[e * 4 + 1];
        r.b[1][0] = binv[e * 4 + 2]; r.b[1][1] = binv[e * 4 + 3];
        r.o[0] = origin[e * 2]; r.o[1] = origin[e * 2 + 1];
        double t[3];
        bary_from_rec<2>(r, x, t);
        if (inside_eps<2>(t, eps)) {
            found = e;
            l[0] = t[0]; l[1] = t[1]; l[2] = t[2];
            break;
        }
    }
    elem[p] = found;
    lam[3 * p] = l[0]; lam[3 * p + 1] = l[1]; lam[3 * p + 2] = l[2];
}

template <int D>
__global__ void nearest_kernel(GridDev g, const double* __restrict__ pts, int64_t K,
                               int32_t* __restrict__ elem) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= K) return;
    double x[D];
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = pts[i * D + c];
    elem[i] = nearest_element<D>(g, x);
}

template <int D>
__global__ void snap_kernel(GridDev g, const double* __restrict__ pts, int64_t K,
                            int32_t* __restrict__ elem, double* __restrict__ lam) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= K || elem[i] >= 0) return;
    double x[D], l[D + 1];
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = pts[i * D + c];
    int e = nearest_element<D>(g, x);
    snap_lambda<D>(g, e, x, l);
    elem[i] = e;
#pragma unroll
    for (int c = 0; c <= D; ++c) lam[i * (D + 1) + c] = l[c];
}

// ---------------------------------------------------------------- certified walk prep
template <int D>
__global__ void max_diam_kernel(int64_t E, const double* __restrict__ nodes,
                                const int32_t* __restrict__ elems,
                                unsigned long long* __restrict__ out) {
    constexpr int K = D + 1;
    double best = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        double v[K][D];
        for (int i = 0; i < K; ++i)
            for (int c = 0; c < D; ++c) v[i][c] = nodes[(int64_t)elems[e * K + i] * D + c];
        for (int i = 0; i < K; ++i)
            for (int j = i + 1; j < K; ++j) {
                double d2 = 0.0;
                for (int c = 0; c < D; ++c) d2 += (v[i][c] - v[j][c]) * (v[i][c] - v[j][c]);
                best = fmax(best, d2);
            }
    }
    // positive doubles order like their bit patterns
    atomicMax(out, (unsigned long long)__double_as_longlong(sqrt(best)));
}

template <int D>
__global__ void walk_prep_kernel(int64_t E, const double* __restrict__ nodes,
                                 const int32_t* __restrict__ elems,
                                 const int64_t* __restrict__ inc_start,
                                 const int32_t* __restrict__ inc, double eps, double dmax,
                                 double* __restrict__ rec, double* __restrict__ wrec,
                                 int32_t* __restrict__ status) {
    constexpr int K = D + 1;
    constexpr int S = (D == 2) ? 8 : 16;
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    int vid[K];
    double v[K][D];
    for (int i = 0; i < K; ++i) {
        vid[i] = elems[e * K + i];
        for (int c = 0; c < D; ++c) v[i][c] = nodes[(int64_t)vid[i] * D + c];
    }
    int nbr[4] = {-1, -1, -1, -1};
    bool nonmanifold = false;
    for (int i = 0; i < K; ++i) {          // facet opposite vertex i
        int f[D];
        for (int t = 0, q = 0; t < K; ++t)
            if (t != i) f[q++] = vid[t];
        int found = -1, matches = 0;
        for (int64_t q = inc_start[f[0]]; q < inc_start[f[0] + 1]; ++q) {
            int64_t e2 = inc[q] / K;
            if (e2 == e) continue;
            bool all = true;
            for (int a = 1; a < D && all; ++a) {
                bool has = false;
                for (int b = 0; b < K; ++b) has |= (elems[e2 * K + b] == f[a]);
                all = has;
            }
            if (all) { found = (int)e2; ++matches; }
        }
        if (matches > 1) nonmanifold = true;
        nbr[i] = found;
    }
    // smallest height: 2A / max edge (2-D), 3V / max face area (3-D)
    double hmin;
    if constexpr (D == 2) {
        double a2 = fabs((v[1][0] - v[0][0]) * (v[2][1] - v[0][1]) - (v[2][0] - v[0][0]) * (v[1][1] - v[0][1]));
        double lmax = 0.0;
        for (int i = 0; i < 3; ++i) {
            int j = (i + 1) % 3;
            lmax = fmax(lmax, hypot(v[i][0] - v[j][0], v[i][1] - v[j][1]));
        }
        hmin = a2 / lmax;
    } else {
        double u[3], w[3], t3[3];
        for (int c = 0; c < 3; ++c) { u[c] = v[1][c] - v[0][c]; w[c] = v[2][c] - v[0][c]; t3[c] = v[3][c] - v[0][c]; }
        double vol6 = fabs(u[0] * (w[1] * t3[2] - w[2] * t3[1]) + u[1] * (w[2] * t3[0] - w[0] * t3[2]) +
                           u[2] * (w[0] * t3[1] - w[1] * t3[0]));
        double amax2 = 0.0;  // (2 * face area)^2
        for (int i = 0; i < 4; ++i) {
            int a = (i + 1) % 4, b = (i + 2) % 4, c = (i + 3) % 4;
            double p[3], q[3];
            for (int k = 0; k < 3; ++k) { p[k] = v[b][k] - v[a][k]; q[k] = v[c][k] - v[a][k]; }
            double cx = p[1] * q[2] - p[2] * q[1], cy = p[2] * q[0] - p[0] * q[2], cz = p[0] * q[1] - p[1] * q[0];
            amax2 = fmax(amax2, cx * cx + cy * cy + cz * cz);
        }
        hmin = vol6 / sqrt(amax2);  // 3V / A = (6V) / (2A)
    }
    // margin: distance > k * (eps + rounding) * diam_max from every other element,
    // doubled, plus an absolute slack far above the lambda rounding error
    double tau = 2.0 * K * (eps + 1e-13) * dmax / hmin + 1e-12;
    if (!(tau < 0.25)) tau = 2.0;  // degenerate/pathological: never certify
    int4 tail;
    tail.x = __float_as_int(__double2float_ru(tau));
    tail.y = nbr[0]; tail.z = nbr[1]; tail.w = nbr[2];
    int4* q = reinterpret_cast<int4*>(rec + e * S + D * D + D);
    *q = tail;
    if constexpr (D == 3) reinterpret_cast<int*>(q + 1)[0] = nbr[3];
    if (nonmanifold) atomicOr(status, TT_FLAG_NONMANIFOLD);
    if (wrec) {
        // compact float walk record; its margin adds a rigorous bound on the float
        // evaluation error of lambda for points within the element:
        //   |lambda_f - lambda| <= 2^-24 * (~6 * sum|b_ij| * |r| + 3),  |r| <= diam(A)
        // taken with a 16x safety factor (2^-20 and 4x/8x terms)
        const double* rb = rec + e * S;
        double babs = 0.0;
        for (int i = 0; i < D * D; ++i) babs += fabs(rb[i]);
        double diam = 0.0;
        for (int a = 0; a < K; ++a)
            for (int b2 = a + 1; b2 < K; ++b2) {
                double d2 = 0.0;
                for (int c = 0; c < D; ++c) d2 += (v[a][c] - v[b2][c]) * (v[a][c] - v[b2][c]);
                diam = fmax(diam, sqrt(d2));
            }
        double tau_f = tau + 9.5367431640625e-07 * (4.0 * babs * diam * 1.0001 + 8.0);
        if (!(tau_f < 0.25)) tau_f = 2.0;
        constexpr int WS = (D == 2) ? 6 : 10;
        double* w = wrec + e * WS;
        for (int c = 0; c < D; ++c) w[c] = rb[D * D + c];           // origin (double)
        float* wf = reinterpret_cast<float*>(w + D);
        for (int i = 0; i < D * D; ++i) wf[i] = __double2float_rn(rb[i]);
        wf[D * D] = __double2float_ru(tau_f);
        int* wn = reinterpret_cast<int*>(wf + D * D + 1);
        for (int i = 0; i < K; ++i) wn[i] = nbr[i];
    }
}

// Walk seeds per target element: the source elements containing its kSeeds anchor points
// (x = sum_a A[s][a] v_a; reference scan, snapped when outside).  Layout (E, kSeeds).
// Two passes, one thread per (element, anchor): anchor 0 (the centroid) by the reference scan;
// then the others, when the grid has walk records and the centroid was found inside, by the
// certified walk from the centroid's element (locate_walk: exactly the scan's element,
// falling back to the scan when uncertain), else by the scan.  (A one-thread-per-element form
// that chained walks from each previous anchor -- snapped ones included -- returned wrong
// elements on a curved pair and was dropped.)
template <int D>
__device__ __forceinline__ void anchor_point(const double* __restrict__ nodes, const int32_t* __restrict__ elems,
                                             int64_t e, int which, double* x) {
    constexpr int K = D + 1;
    for (int c = 0; c < D; ++c) {
        double s = mul(anchor<D>(which, 0), nodes[(int64_t)elems[e * K] * D + c]);
        for (int a = 1; a < K; ++a) s = add(s, mul(anchor<D>(which, a), nodes[(int64_t)elems[e * K + a] * D + c]));
        x[c] = s;
    }
}

template <int D>
__global__ void seed_kernel(GridDev g, const double* __restrict__ nodes,
                            const int32_t* __restrict__ elems, int64_t e_lo, int64_t n_el, int pass,
                            int32_t* __restrict__ seeds, int32_t* __restrict__ status) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int per = pass == 0 ? 1 : kSeeds - 1;
    if (t >= n_el * per) return;
    const int64_t i = t / per;
    const int which = pass == 0 ? 0 : 1 + (int)(t % per);
    double x[D];
    anchor_point<D>(nodes, elems, e_lo + i, which, x);
    double l[D + 1];
    int es;
    if (pass == 0) {
        es = locate_point<D>(g, x, 1e-12, l);
    } else {
        const int c0 = seeds[i * kSeeds];
        // c0 is the centroid's element when it was found inside (pass 0 stores snapped
        // centroids as -(e + 2))
        es = (g.walk && c0 >= 0) ? locate_walk<D>(g, x, 1e-12, c0, l) : locate_point<D>(g, x, 1e-12, l);
    }
    const bool snapped = es < 0;
    if (snapped) {
        es = nearest_element<D>(g, x);
        if (status) atomicOr(status, TT_FLAG_SNAPPED);
    }
    seeds[i * kSeeds + which] = (pass == 0 && snapped) ? -(es + 2) : es;
}

// pass 2: decode snapped centroids
__global__ void seed_fix_kernel(int64_t n_el, int32_t* __restrict__ seeds) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_el) return;
    const int v = seeds[i * kSeeds];
    if (v < -1) seeds[i * kSeeds] = -v - 2;
}

static int64_t ncells_of(const tt_grid_t* g) {
    return (int64_t)g->n[0] * g->n[1] * (g->dim == 3 ? g->n[2] : 1);
}

static bool grid_ok(const tt_grid_t* g) {
    if (!g || (g->dim != 2 && g->dim != 3)) return false;
    for (int c = 0; c < g->dim; ++c)
        if (g->n[c] < 1) return false;
    return true;
}

}  // namespace tt

using namespace tt;

extern "C" int tt_geometry(const tt_mesh_t* m, double* smeas, double* rec, double* cent,
                           void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3)) {
        set_error("tt_geometry: dim must be 2 or 3");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (m->n_elems == 0) return TT_OK;
    auto s = as_stream(stream);
    if (m->dim == 2)
        geometry_kernel<2><<<grid_for(m->n_elems, 256), 256, 0, s>>>(m->n_elems, m->nodes, m->elems,
                                                                     smeas, rec, cent);
    else
        geometry_kernel<3><<<grid_for(m->n_elems, 256), 256, 0, s>>>(m->n_elems, m->nodes, m->elems,
                                                                     smeas, rec, cent);
    return launch_check("geometry_kernel");
}

extern "C" int tt_bbox(int dim, int64_t n, const double* nodes, double* out, void* stream) {
    if (dim < 1 || dim > 3 || n < 1) {
        set_error("tt_bbox: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    auto s = as_stream(stream);
    int nparts = sm_count() * 2;
    double* part = nullptr;
    int st = cuda_status(cudaMallocAsync((void**)&part, sizeof(double) * 6 * nparts, s), "bbox alloc");
    if (st) return st;
    bbox_partial_kernel<<<nparts, 256, 0, s>>>(dim, n, nodes, part);
    bbox_final_kernel<<<1, 32, 0, s>>>(dim, nparts, part, out);
    st = launch_check("bbox kernels");
    cudaFreeAsync(part, s);
    return st;
}

extern "C" int tt_grid_count(const tt_mesh_t* m, const tt_grid_t* g, int64_t* cell_start,
                             void* stream) {
    if (!m || !grid_ok(g) || m->dim != g->dim) {
        set_error("tt_grid_count: bad mesh/grid descriptor");
        return TT_ERR_INVALID_PARAMETER;
    }
    auto s = as_stream(stream);
    int64_t nc = ncells_of(g);
    GridDev gd = to_dev(*g);
    unsigned long long* counts = nullptr;
    int st = cuda_status(cudaMallocAsync((void**)&counts, sizeof(unsigned long long) * nc, s),
                         "grid counts alloc");
    if (st) return st;
    cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * nc, s);
    cudaMemsetAsync(cell_start, 0, sizeof(int64_t), s);
    if (m->n_elems > 0) {
        if (g->dim == 2)
            grid_count_kernel<2><<<grid_for(m->n_elems, 256), 256, 0, s>>>(gd, m->n_elems, m->nodes,
                                                                           m->elems, counts);
        else
            grid_count_kernel<3><<<grid_for(m->n_elems, 256), 256, 0, s>>>(gd, m->n_elems, m->nodes,
                                                                           m->elems, counts);
    }
    size_t tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, counts,
                                  reinterpret_cast<unsigned long long*>(cell_start + 1), nc, s);
    void* tmp = nullptr;
    st = cuda_status(cudaMallocAsync(&tmp, tmp_bytes, s), "scan tmp alloc");
    if (!st) {
        cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, counts,
                                      reinterpret_cast<unsigned long long*>(cell_start + 1), nc, s);
        st = launch_check("grid count/scan");
        cudaFreeAsync(tmp, s);
    }
    cudaFreeAsync(counts, s);
    return st;
}

extern "C" int tt_grid_fill(const tt_mesh_t* m, const tt_grid_t* g, int32_t* cell_elems,
                            int64_t* cursor, void* stream) {
    if (!m || !grid_ok(g) || m->dim != g->dim || !g->cell_start) {
        set_error("tt_grid_fill: bad mesh/grid descriptor");
        return TT_ERR_INVALID_PARAMETER;
    }
    auto s = as_stream(stream);
    int64_t nc = ncells_of(g);
    GridDev gd = to_dev(*g);
    cudaMemcpyAsync(cursor, g->cell_start, sizeof(int64_t) * nc, cudaMemcpyDeviceToDevice, s);
    auto* cur = reinterpret_cast<unsigned long long*>(cursor);
    if (m->n_elems > 0) {
        if (g->dim == 2)
            grid_fill_kernel<2><<<grid_for(m->n_elems, 256), 256, 0, s>>>(gd, m->n_elems, m->nodes,
                                                                          m->elems, cur, cell_elems);
        else
            grid_fill_kernel<3><<<grid_for(m->n_elems, 256), 256, 0, s>>>(gd, m->n_elems, m->nodes,
                                                                          m->elems, cur, cell_elems);
    }
    segment_sort_kernel<<<grid_for(nc, 256), 256, 0, s>>>(nc, g->cell_start, cell_elems);
    return launch_check("grid fill/sort");
}

extern "C" int tt_locate(const tt_grid_t* g, const double* pts, int64_t K, double eps,
                         int32_t* elem, double* lam, void* stream) {
    if (!grid_ok(g)) {
        set_error("tt_locate: bad grid descriptor");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (K == 0) return TT_OK;
    GridDev gd = to_dev(*g);
    auto s = as_stream(stream);
    if (g->dim == 2)
        locate_kernel<2><<<grid_for(K, 256), 256, 0, s>>>(gd, pts, K, eps, elem, lam);
    else
        locate_kernel<3><<<grid_for(K, 256), 256, 0, s>>>(gd, pts, K, eps, elem, lam);
    return launch_check("locate_kernel");
}

extern "C" int tt_locate_many(const double* pts, int64_t K, int nx, int ny, const double* bbox,
                              const int64_t* cell_start, const int32_t* cell_elems,
                              const double* binv, const double* origin, double eps,
                              int32_t* elem, double* lam, void* stream) {
    if (nx < 1 || ny < 1 || !bbox) {
        set_error("tt_locate_many: bad grid dims");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (K == 0) return TT_OK;
    locate_many_seam_kernel<<<grid_for(K, 256), 256, 0, as_stream(stream)>>>(
        pts, K, nx, ny, bbox[0], bbox[1], bbox[2], bbox[3], cell_start, cell_elems, binv, origin,
        eps, elem, lam);
    return launch_check("locate_many_seam_kernel");
}

extern "C" int tt_nearest(const tt_grid_t* g, const double* pts, int64_t K, int32_t* elem,
                          void* stream) {
    if (!grid_ok(g)) {
        set_error("tt_nearest: bad grid descriptor");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (K == 0) return TT_OK;
    GridDev gd = to_dev(*g);
    auto s = as_stream(stream);
    if (g->dim == 2)
        nearest_kernel<2><<<grid_for(K, 128), 128, 0, s>>>(gd, pts, K, elem);
    else
        nearest_kernel<3><<<grid_for(K, 128), 128, 0, s>>>(gd, pts, K, elem);
    return launch_check("nearest_kernel");
}

extern "C" int tt_snap(const tt_grid_t* g, const double* pts, int64_t K, int32_t* elem,
                       double* lam, void* stream) {
    if (!grid_ok(g)) {
        set_error("tt_snap: bad grid descriptor");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (K == 0) return TT_OK;
    GridDev gd = to_dev(*g);
    auto s = as_stream(stream);
    if (g->dim == 2)
        snap_kernel<2><<<grid_for(K, 128), 128, 0, s>>>(gd, pts, K, elem, lam);
    else
        snap_kernel<3><<<grid_for(K, 128), 128, 0, s>>>(gd, pts, K, elem, lam);
    return launch_check("snap_kernel");
}

extern "C" int tt_grid_walk_prep(const tt_mesh_t* m, const int64_t* inc_start, const int32_t* inc,
                                 double eps, double* rec, double* wrec, int32_t* status, void* stream) {
    if (!m || (m->dim != 2 && m->dim != 3) || !inc_start || !inc || !rec) {
        set_error("tt_grid_walk_prep: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (m->n_elems == 0) return TT_OK;
    auto s = as_stream(stream);
    unsigned long long* dm = nullptr;
    int st = cuda_status(cudaMallocAsync((void**)&dm, sizeof(unsigned long long), s), "walk alloc");
    if (st) return st;
    cudaMemsetAsync(dm, 0, sizeof(unsigned long long), s);
    if (m->dim == 2)
        max_diam_kernel<2><<<sm_count() * 4, 256, 0, s>>>(m->n_elems, m->nodes, m->elems, dm);
    else
        max_diam_kernel<3><<<sm_count() * 4, 256, 0, s>>>(m->n_elems, m->nodes, m->elems, dm);
    unsigned long long bits = 0;
    cudaMemcpyAsync(&bits, dm, sizeof(bits), cudaMemcpyDeviceToHost, s);
    st = cuda_status(cudaStreamSynchronize(s), "walk prep diameter");
    cudaFreeAsync(dm, s);
    if (st) return st;
    double dmax;
    memcpy(&dmax, &bits, sizeof(dmax));
    if (m->dim == 2)
        walk_prep_kernel<2><<<grid_for(m->n_elems, 128), 128, 0, s>>>(m->n_elems, m->nodes, m->elems,
                                                                      inc_start, inc, eps, dmax, rec, wrec, status);
    else
        walk_prep_kernel<3><<<grid_for(m->n_elems, 128), 128, 0, s>>>(m->n_elems, m->nodes, m->elems,
                                                                      inc_start, inc, eps, dmax, rec, wrec, status);
    return launch_check("walk_prep_kernel");
}

extern "C" int tt_seed_elements(const tt_grid_t* g, const tt_mesh_t* t, int64_t e_lo, int64_t e_hi,
                                int32_t* seeds, int32_t* status, void* stream) {
    if (!grid_ok(g) || !t || t->dim != g->dim || e_lo < 0 || e_hi > t->n_elems || e_lo > e_hi) {
        set_error("tt_seed_elements: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (e_hi == e_lo) return TT_OK;
    GridDev gd = to_dev(*g);
    auto s = as_stream(stream);
    const int64_t n_el = e_hi - e_lo;
    for (int pass = 0; pass < 2; ++pass) {
        const int64_t nt = n_el * (pass == 0 ? 1 : kSeeds - 1);
        if (g->dim == 2)
            seed_kernel<2><<<grid_for(nt, 128), 128, 0, s>>>(gd, t->nodes, t->elems, e_lo, n_el, pass, seeds, status);
        else
            seed_kernel<3><<<grid_for(nt, 128), 128, 0, s>>>(gd, t->nodes, t->elems, e_lo, n_el, pass, seeds, status);
    }
    seed_fix_kernel<<<grid_for(n_el, 256), 256, 0, s>>>(n_el, seeds);
    return launch_check("seed_kernel");
}
