// Supermesh error metrics for P1 fields on two triangle meshes (metrics.py:35-74; the
// intersection polygons of intersect.py:60-80 / _pure.py:13-62, clipped on the fly).
//
// One thread per target element t: the source elements whose bounding-box cells overlap
// t's (the source's uniform grid, each candidate visited once: in the first cell common to
// both boxes), each clipped against t with the reference's Sutherland-Hodgman loop
// (half-planes of t's edges in order, same predicate and intersection formula, the same
// near-duplicate removal), polygons of area <= SLIVER_REL |t| dropped (intersect.py:21,79).
// Both fields are linear on every polygon, so the integrals over its fan from vertex 0 are
// closed forms of the vertex values (exact, as the reference's degree-2 rule):
//   int f = A (fa + fb + fc) / 3,   int f^2 = A (fa^2 + fb^2 + fc^2 + fa fb + fb fc + fc fa) / 6.
// Per target element: int (fs - ft)^2, int fs^2, int fs, int ft and the covered area; the
// totals are reduced in a fixed order (deterministic).
#include "tt_common.cuh"

namespace tt {

constexpr int kMaxPoly = 9;

struct Tri2 {
    double x[3], y[3];
};

// Sutherland-Hodgman clip of the vertex loop (px, py, n) against the CCW half-planes of t,
// in the reference's order and arithmetic (_pure.py:25-49), then _dedupe (:52-62).
__device__ int clip_poly(const Tri2& t, double* px, double* py, int n) {
    double ox[kMaxPoly], oy[kMaxPoly];
    for (int k = 0; k < 3 && n > 0; ++k) {
        const double ax = t.x[k], ay = t.y[k];
        const double ex = sub(t.x[(k + 1) % 3], ax), ey = sub(t.y[(k + 1) % 3], ay);
        int m = 0;
        double qx0 = px[n - 1], qy0 = py[n - 1];
        double dp = sub(mul(ex, sub(qy0, ay)), mul(ey, sub(qx0, ax)));
        for (int i = 0; i < n; ++i) {
            const double qx = px[i], qy = py[i];
            const double dq = sub(mul(ex, sub(qy, ay)), mul(ey, sub(qx, ax)));
            if (dq >= 0.0) {
                if (dp < 0.0) {
                    const double f = div(dp, sub(dp, dq));
                    ox[m] = add(qx0, mul(f, sub(qx, qx0))); oy[m] = add(qy0, mul(f, sub(qy, qy0))); ++m;
                }
                ox[m] = qx; oy[m] = qy; ++m;
            } else if (dp >= 0.0) {
                const double f = div(dp, sub(dp, dq));
                ox[m] = add(qx0, mul(f, sub(qx, qx0))); oy[m] = add(qy0, mul(f, sub(qy, qy0))); ++m;
            }
            qx0 = qx; qy0 = qy; dp = dq;
        }
        n = m;
        for (int i = 0; i < n; ++i) { px[i] = ox[i]; py[i] = oy[i]; }
    }
    if (n < 2) return n;
    double scale = 0.0;
    for (int i = 0; i < n; ++i) scale = fmax(scale, add(fabs(px[i]), fabs(py[i])));
    const double lim = 1e-24 * (scale * scale + 1e-300);  // rel * scale2 (_pure.py:55)
    int m = 0;
    for (int i = 0; i < n; ++i) {
        if (m == 0) { px[m] = px[i]; py[m] = py[i]; ++m; continue; }
        const double dx = sub(px[i], px[m - 1]), dy = sub(py[i], py[m - 1]);
        if (add(mul(dx, dx), mul(dy, dy)) > lim) { px[m] = px[i]; py[m] = py[i]; ++m; }
    }
    while (m > 1) {
        const double dx = sub(px[0], px[m - 1]), dy = sub(py[0], py[m - 1]);
        if (add(mul(dx, dx), mul(dy, dy)) <= lim) --m;
        else break;
    }
    return m;
}

__device__ __forceinline__ double p1_at(const Tri2& v, const double* c, double x, double y) {
    // barycentrics of (x, y) in v (origin v2, mesh.py:140-159), then sum c_i lambda_i
    const double d0x = v.x[0] - v.x[2], d0y = v.y[0] - v.y[2];
    const double d1x = v.x[1] - v.x[2], d1y = v.y[1] - v.y[2];
    const double det = d0x * d1y - d1x * d0y;
    const double rx = x - v.x[2], ry = y - v.y[2];
    const double l0 = (d1y * rx - d1x * ry) / det;
    const double l1 = (-d0y * rx + d0x * ry) / det;
    const double l2 = 1.0 - l0 - l1;
    return c[0] * l0 + c[1] * l1 + c[2] * l2;
}

__global__ void supermesh_kernel(int64_t E_t, const double* __restrict__ t_nodes, const int32_t* __restrict__ t_elems,
                                 const double* __restrict__ t_coeffs, GridDev g,
                                 const double* __restrict__ s_nodes, const int32_t* __restrict__ s_elems,
                                 const double* __restrict__ s_coeffs, double sliver_rel,
                                 double* __restrict__ out /* (E_t, 6) */) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E_t) return;
    Tri2 t;
    double ct[3];
    for (int i = 0; i < 3; ++i) {
        const int n = t_elems[e * 3 + i];
        t.x[i] = t_nodes[2 * (int64_t)n];
        t.y[i] = t_nodes[2 * (int64_t)n + 1];
        ct[i] = t_coeffs[n];
    }
    const double area_t = 0.5 * fabs(sub(mul(sub(t.x[1], t.x[0]), sub(t.y[2], t.y[0])),
                                         mul(sub(t.x[2], t.x[0]), sub(t.y[1], t.y[0]))));
    const double eps_area = sliver_rel * area_t;
    const double tx0 = fmin(fmin(t.x[0], t.x[1]), t.x[2]), tx1 = fmax(fmax(t.x[0], t.x[1]), t.x[2]);
    const double ty0 = fmin(fmin(t.y[0], t.y[1]), t.y[2]), ty1 = fmax(fmax(t.y[0], t.y[1]), t.y[2]);
    const int cx0 = axis_cell(tx0, g.lo[0], g.hi[0], g.n0), cx1 = axis_cell(tx1, g.lo[0], g.hi[0], g.n0);
    const int cy0 = axis_cell(ty0, g.lo[1], g.hi[1], g.n1), cy1 = axis_cell(ty1, g.lo[1], g.hi[1], g.n1);
    double s_g2 = 0.0, s_fs2 = 0.0, s_fs = 0.0, s_ft = 0.0, s_area = 0.0;
    for (int cx = cx0; cx <= cx1; ++cx)
        for (int cy = cy0; cy <= cy1; ++cy) {
            const int64_t c = (int64_t)cx * g.n1 + cy;
            for (int64_t j = g.cell_start[c]; j < g.cell_start[c + 1]; ++j) {
                const int s = g.cell_elems[j];
                Tri2 v;
                double cs[3];
                for (int i = 0; i < 3; ++i) {
                    const int n = s_elems[(int64_t)s * 3 + i];
                    v.x[i] = s_nodes[2 * (int64_t)n];
                    v.y[i] = s_nodes[2 * (int64_t)n + 1];
                    cs[i] = s_coeffs[n];
                }
                // visit s once: in the first cell common to both bounding boxes
                const double sx0 = fmin(fmin(v.x[0], v.x[1]), v.x[2]);
                const double sy0 = fmin(fmin(v.y[0], v.y[1]), v.y[2]);
                const int fx = max(cx0, axis_cell(sx0, g.lo[0], g.hi[0], g.n0));
                const int fy = max(cy0, axis_cell(sy0, g.lo[1], g.hi[1], g.n1));
                if (fx != cx || fy != cy) continue;
                double px[kMaxPoly], py[kMaxPoly];
                for (int i = 0; i < 3; ++i) { px[i] = v.x[i]; py[i] = v.y[i]; }
                const int n = clip_poly(t, px, py, 3);
                if (n < 3) continue;
                double a2 = 0.0;  // shoelace in clip order (ConvexPolygon.area)
                for (int i = 0; i < n; ++i) {
                    const int k = (i + 1) % n;
                    a2 += px[i] * py[k] - px[k] * py[i];
                }
                if (0.5 * a2 <= eps_area) continue;
                double fs[kMaxPoly], ft[kMaxPoly];
                for (int i = 0; i < n; ++i) {
                    fs[i] = p1_at(v, cs, px[i], py[i]);
                    ft[i] = p1_at(t, ct, px[i], py[i]);
                }
                for (int i = 1; i + 1 < n; ++i) {
                    const double A = 0.5 * ((px[i] - px[0]) * (py[i + 1] - py[0]) - (px[i + 1] - px[0]) * (py[i] - py[0]));
                    const double a = fs[0], b = fs[i], cc = fs[i + 1];
                    const double u = ft[0], w = ft[i], z = ft[i + 1];
                    const double ga = a - u, gb = b - w, gc = cc - z;
                    s_fs += A * (a + b + cc) / 3.0;
                    s_ft += A * (u + w + z) / 3.0;
                    s_fs2 += A * (a * a + b * b + cc * cc + a * b + b * cc + cc * a) / 6.0;
                    s_g2 += A * (ga * ga + gb * gb + gc * gc + ga * gb + gb * gc + gc * ga) / 6.0;
                    s_area += A;
                }
            }
        }
    double* o = out + e * 6;
    o[0] = s_g2; o[1] = s_fs2; o[2] = s_fs; o[3] = s_ft; o[4] = s_area;
    o[5] = s_area / area_t;
}

// totals[0..5) = column sums of out in element order (per-block partials, then one block
// in block order); totals[5] = min covered fraction
__global__ void super_partials_kernel(int64_t E, const double* __restrict__ per, double* __restrict__ part) {
    __shared__ double sh[6][256];
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 2.0};
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        for (int k = 0; k < 5; ++k) acc[k] += per[e * 6 + k];
        acc[5] = fmin(acc[5], per[e * 6 + 5]);
    }
    for (int k = 0; k < 6; ++k) sh[k][threadIdx.x] = acc[k];
    __syncthreads();
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        double t = k == 5 ? 2.0 : 0.0;
        for (int i = 0; i < (int)blockDim.x; ++i) t = k == 5 ? fmin(t, sh[k][i]) : t + sh[k][i];
        part[blockIdx.x * 6 + k] = t;
    }
}

__global__ void super_totals_kernel(int nb, const double* __restrict__ part, double* __restrict__ totals) {
    const int k = threadIdx.x;
    if (k >= 6) return;
    double t = k == 5 ? 2.0 : 0.0;
    for (int b = 0; b < nb; ++b) t = k == 5 ? fmin(t, part[b * 6 + k]) : t + part[b * 6 + k];
    totals[k] = t;
}

}  // namespace tt

using namespace tt;

extern "C" int tt_supermesh_integrals(const tt_mesh_t* target, const double* t_coeffs,
                                      const tt_mesh_t* source, const double* s_coeffs,
                                      const tt_grid_t* src_grid, double sliver_rel,
                                      double* per_elem, double* totals, void* stream) {
    if (!target || !source || !src_grid || target->dim != 2 || source->dim != 2 || src_grid->dim != 2 ||
        !t_coeffs || !s_coeffs || !per_elem || !totals) {
        set_error("tt_supermesh_integrals: 2-D meshes, coefficients and outputs required");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (target->n_elems == 0) return TT_OK;
    auto s = as_stream(stream);
    supermesh_kernel<<<grid_for(target->n_elems, 128), 128, 0, s>>>(
        target->n_elems, target->nodes, target->elems, t_coeffs, to_dev(*src_grid), source->nodes,
        source->elems, s_coeffs, sliver_rel, per_elem);
    const int nb = 148;
    double* part = nullptr;
    int st = cuda_status(cudaMallocAsync((void**)&part, sizeof(double) * 6 * nb, s), "supermesh alloc");
    if (st) return st;
    super_partials_kernel<<<nb, 256, 0, s>>>(target->n_elems, per_elem, part);
    super_totals_kernel<<<1, 32, 0, s>>>(nb, part, totals);
    st = launch_check("supermesh kernels");
    cudaFreeAsync(part, s);
    return st;
}
