/* CPU port of the reference Monte-Carlo load (mesh-backed source), d = 2, 3.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY: used by tests/ (as a checker, against the numpy
 * oracle) and by bench.py's cpu_baseline / --impl reference legs.  The product never
 * links it.  It restates, in plain C with OpenMP over the reference's fixed 512-element
 * chunk grid (montecarlo.py:17,186-200):
 *   point map            montecarlo.py:123-124     x = ((l0 v0 + l1 v1) + l2 v2) [+ l3 v3]
 *   grid locate          _compiled.pyx:147-174     first ascending candidate, lambda >= -eps
 *   nearest + snap       locate.py:97-127, montecarlo.py:58-63
 *   P1 evaluation        fem.py:36-38
 *   accumulate           montecarlo.py:128-131     contrib[e,a] += f/(N p) * lam_a, p = 1/|T|
 *   grid build           locate.py:42-70           every element into each cell its bbox overlaps,
 *                                                  ascending ids per cell (counting sort = the
 *                                                  reference's stable argsort)
 * Compile: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no FMA: bit-exact ids).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
    int dim, n[3];
    double lo[3], hi[3];
    const int64_t* cell_start;
    const int32_t* cell_elems;
    const double* binv;     /* (E, d, d) */
    const double* origin;   /* (E, d) */
    const double* centroids;/* (E, d) */
} grid_t;

static int axis_cell(double v, double lo, double hi, int n) {
    double t = (v - lo) / (hi - lo) * n;
    int i = (t > -2147483649.0 && t < 2147483648.0) ? (int)t : (int)0x80000000;
    if (i < 0) i = 0;
    if (i > n - 1) i = n - 1;
    return i;
}

static void bary(const grid_t* g, int e, const double* x, double* l) {
    const int d = g->dim;
    const double* b = g->binv + (int64_t)e * d * d;
    const double* o = g->origin + (int64_t)e * d;
    double r[3];
    for (int c = 0; c < d; ++c) r[c] = x[c] - o[c];
    for (int i = 0; i < d; ++i) {
        double acc = b[i * d + 0] * r[0] + b[i * d + 1] * r[1];
        if (d == 3) acc = acc + b[i * d + 2] * r[2];
        l[i] = acc;
    }
    double last = 1.0 - l[0] - l[1];
    if (d == 3) last = last - l[2];
    l[d] = last;
}

static int locate(const grid_t* g, const double* x, double eps, double* lam) {
    const int d = g->dim;
    int ix = axis_cell(x[0], g->lo[0], g->hi[0], g->n[0]);
    int iy = axis_cell(x[1], g->lo[1], g->hi[1], g->n[1]);
    int64_t c = (int64_t)ix * g->n[1] + iy;
    if (d == 3) c = c * g->n[2] + axis_cell(x[2], g->lo[2], g->hi[2], g->n[2]);
    for (int64_t j = g->cell_start[c]; j < g->cell_start[c + 1]; ++j) {
        int e = g->cell_elems[j];
        double l[4];
        bary(g, e, x, l);
        int ok = 1;
        for (int i = 0; i <= d; ++i) ok &= (l[i] >= -eps);
        if (ok) {
            for (int i = 0; i <= d; ++i) lam[i] = l[i];
            return e;
        }
    }
    return -1;
}

static int nearest(const grid_t* g, const double* x) {
    const int d = g->dim;
    int home[3] = {0, 0, 0};
    const int n2 = d == 3 ? g->n[2] : 1;
    const int n[3] = {g->n[0], g->n[1], n2};
    for (int c = 0; c < d; ++c) {
        double t = (x[c] - g->lo[c]) / (g->hi[c] - g->lo[c]) * n[c];
        if (t < 0) t = 0;
        if (t > n[c] - 1) t = n[c] - 1;
        home[c] = (int)t;
    }
    int best = -1, first = -1;
    double best_d2 = INFINITY;
    int max_ring = n[0] > n[1] ? n[0] : n[1];
    if (n[2] > max_ring) max_ring = n[2];
    for (int ring = 0; ring <= max_ring; ++ring) {
        if (first >= 0 && ring > first + 1) break;
        int rz = d == 3 ? ring : 0;
        for (int cx = home[0] - ring; cx <= home[0] + ring; ++cx)
            for (int cy = home[1] - ring; cy <= home[1] + ring; ++cy)
                for (int cz = home[2] - rz; cz <= home[2] + rz; ++cz) {
                    int a = abs(cx - home[0]), b = abs(cy - home[1]), cc = abs(cz - home[2]);
                    int cheb = a > b ? a : b;
                    if (cc > cheb) cheb = cc;
                    if (cheb != ring) continue;
                    if (cx < 0 || cx >= n[0] || cy < 0 || cy >= n[1] || cz < 0 || cz >= n[2]) continue;
                    int64_t cell = ((int64_t)cx * n[1] + cy) * n[2] + cz;
                    for (int64_t j = g->cell_start[cell]; j < g->cell_start[cell + 1]; ++j) {
                        int e = g->cell_elems[j];
                        const double* ce = g->centroids + (int64_t)e * d;
                        double d0 = ce[0] - x[0], d1 = ce[1] - x[1];
                        double d2 = d0 * d0 + d1 * d1;
                        if (d == 3) { double dz = ce[2] - x[2]; d2 = d2 + dz * dz; }
                        if (d2 < best_d2 || (d2 == best_d2 && e < best)) { best = e; best_d2 = d2; }
                        if (first < 0) first = ring;
                    }
                }
    }
    return best;
}

/* contrib (e_hi - e_lo, k); returns the number of OUTSIDE (snapped) samples, or -1
 * if any source value is non-finite. */
int64_t tto_mc_load_mesh(int dim, const double* t_nodes, const int32_t* t_elems,
                         const double* t_measure, int64_t e_lo, int64_t e_hi, int64_t N,
                         const double* lam, const int32_t* s_elems, const double* s_coeffs,
                         const int32_t* gdims, const double* glo, const double* ghi,
                         const int64_t* cell_start, const int32_t* cell_elems,
                         const double* binv, const double* origin, const double* centroids,
                         double eps, double* contrib, int32_t* ids /* (e_hi-e_lo, N) or NULL */,
                         int nthreads) {
    grid_t g;
    g.dim = dim;
    for (int c = 0; c < 3; ++c) { g.n[c] = gdims[c]; g.lo[c] = glo[c]; g.hi[c] = ghi[c]; }
    g.cell_start = cell_start; g.cell_elems = cell_elems;
    g.binv = binv; g.origin = origin; g.centroids = centroids;
    const int k = dim + 1;
    const int64_t chunk = 512;
    const int64_t nchunks = (e_hi - e_lo + chunk - 1) / chunk;
    int64_t outside = 0, bad = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(+:outside, bad)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        int64_t c0 = e_lo + ch * chunk, c1 = c0 + chunk < e_hi ? c0 + chunk : e_hi;
        for (int64_t e = c0; e < c1; ++e) {
            double v[4][3];
            for (int i = 0; i < k; ++i)
                for (int c = 0; c < dim; ++c) v[i][c] = t_nodes[(int64_t)t_elems[e * k + i] * dim + c];
            const double p = 1.0 / t_measure[e];
            double acc[4] = {0, 0, 0, 0};
            for (int64_t j = 0; j < N; ++j) {
                const double* lj = lam + j * k;
                double x[3];
                for (int c = 0; c < dim; ++c) {
                    double s = lj[0] * v[0][c] + lj[1] * v[1][c];
                    s = s + lj[2] * v[2][c];
                    if (dim == 3) s = s + lj[3] * v[3][c];
                    x[c] = s;
                }
                double l[4];
                int es = locate(&g, x, eps, l);
                if (es < 0) {
                    ++outside;
                    es = nearest(&g, x);
                    bary(&g, es, x, l);
                    double sum = 0.0;
                    for (int i = 0; i <= dim; ++i) l[i] = l[i] < 0.0 ? 0.0 : l[i];
                    sum = l[0] + l[1];
                    for (int i = 2; i <= dim; ++i) sum = sum + l[i];
                    for (int i = 0; i <= dim; ++i) l[i] = l[i] / sum;
                }
                if (ids) ids[(e - e_lo) * N + j] = es;
                const int32_t* conn = s_elems + (int64_t)es * k;
                double f = s_coeffs[conn[0]] * l[0];
                for (int i = 1; i < k; ++i) f = f + s_coeffs[conn[i]] * l[i];
                if (!isfinite(f)) ++bad;
                const double w = f / (N * p);
                for (int a = 0; a < k; ++a) acc[a] += w * lj[a];
            }
            for (int a = 0; a < k; ++a) contrib[(e - e_lo) * k + a] = acc[a];
        }
    }
    return bad ? -1 : outside;
}

/* Uniform-grid build (locate.py:42-70), d = 2, 3: per element, the cell range of its
 * vertex bbox (trunc((v - lo)/(hi - lo) * n) with C int semantics, clamped; z outermost
 * last: cell = (ix*n1 + iy)*n2 + iz).  Pass 1 (cell_elems == NULL): counts -> exclusive
 * scan into cell_start (ncell + 1).  Pass 2: fill in ascending element order, which is the
 * order the reference's stable argsort leaves in every cell. */
static void elem_cell_range(int dim, const double* nodes, const int32_t* elems, int64_t e,
                            const int32_t* n, const double* lo, const double* hi, int* c0, int* c1) {
    const int k = dim + 1;
    for (int c = 0; c < 3; ++c) { c0[c] = 0; c1[c] = 0; }
    for (int c = 0; c < dim; ++c) {
        double mn = nodes[(int64_t)elems[e * k] * dim + c], mx = mn;
        for (int i = 1; i < k; ++i) {
            double v = nodes[(int64_t)elems[e * k + i] * dim + c];
            mn = v < mn ? v : mn;   /* np.min / np.max (no NaN in valid meshes) */
            mx = v > mx ? v : mx;
        }
        c0[c] = axis_cell(mn, lo[c], hi[c], n[c]);
        c1[c] = axis_cell(mx, lo[c], hi[c], n[c]);
    }
}

int64_t tto_grid_build(int dim, const double* nodes, const int32_t* elems, int64_t E,
                       const int32_t* gdims, const double* glo, const double* ghi,
                       int64_t* cell_start, int32_t* cell_elems) {
    const int32_t n[3] = {gdims[0], gdims[1], dim == 3 ? gdims[2] : 1};
    const int64_t ncell = (int64_t)n[0] * n[1] * n[2];
    if (!cell_elems) {
        for (int64_t c = 0; c <= ncell; ++c) cell_start[c] = 0;
        for (int64_t e = 0; e < E; ++e) {
            int c0[3], c1[3];
            elem_cell_range(dim, nodes, elems, e, n, glo, ghi, c0, c1);
            for (int ix = c0[0]; ix <= c1[0]; ++ix)
                for (int iy = c0[1]; iy <= c1[1]; ++iy)
                    for (int iz = c0[2]; iz <= c1[2]; ++iz)
                        ++cell_start[((int64_t)ix * n[1] + iy) * n[2] + iz + 1];
        }
        for (int64_t c = 0; c < ncell; ++c) cell_start[c + 1] += cell_start[c];
        return cell_start[ncell];
    }
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncell > 0 ? ncell : 1));
    for (int64_t c = 0; c < ncell; ++c) cur[c] = cell_start[c];
    for (int64_t e = 0; e < E; ++e) {
        int c0[3], c1[3];
        elem_cell_range(dim, nodes, elems, e, n, glo, ghi, c0, c1);
        for (int ix = c0[0]; ix <= c1[0]; ++ix)
            for (int iy = c0[1]; iy <= c1[1]; ++iy)
                for (int iz = c0[2]; iz <= c1[2]; ++iz)
                    cell_elems[cur[((int64_t)ix * n[1] + iy) * n[2] + iz]++] = (int32_t)e;
    }
    free(cur);
    return cell_start[ncell];
}
