/*
 * c_transfer.c -- a complete Monte-Carlo transfer through the C ABI alone (no Python):
 * the reference's transfer_mc(target, MeshBackedField(field), SamplePlan.build(N, "sobol", 0))
 * (transfer.py:158-163) on two structured unit-square triangle meshes.
 *
 *   gcc -O2 -std=c11 examples/c_transfer.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2603_00538_b200 -ltt_b200 -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -lpthread -lm \
 *       -Wl,-rpath,$PWD/paper_2603_00538_b200 -o examples/c_transfer
 *   ./examples/c_transfer 12 16 256        # target n, source n, samples per element
 *
 * Prints the transferred field's integral, the solve's iteration count and a checksum;
 * tests/test_gpu_api.py compares them with the Python API on the same inputs.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "tt_b200.h"

#define CK(x)                                                                              \
    do {                                                                                   \
        int _s = (x);                                                                      \
        if (_s) {                                                                          \
            fprintf(stderr, "%s failed (%d): %s\n", #x, _s, tt_last_error());              \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)
#define CU(x)                                                                              \
    do {                                                                                   \
        cudaError_t _e = (x);                                                              \
        if (_e != cudaSuccess) {                                                           \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(_e));                       \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

/* structured unit square, "left" diagonals, no jitter: (n+1)^2 nodes, 2n^2 CCW triangles */
static void square_mesh(int n, double** nodes, int32_t** elems, int64_t* nn, int64_t* ne) {
    *nn = (int64_t)(n + 1) * (n + 1);
    *ne = 2LL * n * n;
    *nodes = malloc(sizeof(double) * 2 * *nn);
    *elems = malloc(sizeof(int32_t) * 3 * *ne);
    for (int i = 0; i <= n; ++i)
        for (int j = 0; j <= n; ++j) {
            (*nodes)[2 * (i * (n + 1) + j)] = (double)i * (1.0 / n);   /* numpy linspace */
            (*nodes)[2 * (i * (n + 1) + j) + 1] = (double)j * (1.0 / n);
        }
    int64_t t = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            int v00 = i * (n + 1) + j, v10 = (i + 1) * (n + 1) + j, v01 = v00 + 1, v11 = v10 + 1;
            int32_t a[6] = {v00, v10, v11, v00, v11, v01};
            for (int q = 0; q < 6; ++q) (*elems)[3 * t + q] = a[q];
            t += 2;
        }
}

static void* dup(const void* h, size_t bytes) {
    void* d;
    CU(cudaMalloc(&d, bytes ? bytes : 1));
    if (bytes) CU(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
    return d;
}

int main(int argc, char** argv) {
    const int nt = argc > 1 ? atoi(argv[1]) : 12, ns = argc > 2 ? atoi(argv[2]) : 16;
    const int64_t N = argc > 3 ? atoll(argv[3]) : 256;
    void* st = NULL;  /* legacy default stream */
    double *tn, *sn;
    int32_t *te, *se;
    int64_t tnn, tne, snn, sne;
    square_mesh(nt, &tn, &te, &tnn, &tne);
    square_mesh(ns, &sn, &se, &snn, &sne);

    /* device meshes + geometry (|measure|, packed locate records, centroids) */
    tt_mesh_t T = {2, 0, tnn, tne, dup(tn, 16 * tnn), dup(te, 12 * tne), NULL};
    tt_mesh_t S = {2, 0, snn, sne, dup(sn, 16 * snn), dup(se, 12 * sne), NULL};
    double *tmeas, *smeas, *srec, *scent, *trec, *tcent;
    CU(cudaMalloc((void**)&tmeas, 8 * tne)); CU(cudaMalloc((void**)&smeas, 8 * sne));
    CU(cudaMalloc((void**)&trec, 64 * tne)); CU(cudaMalloc((void**)&tcent, 16 * tne));
    CU(cudaMalloc((void**)&srec, 64 * sne)); CU(cudaMalloc((void**)&scent, 16 * sne));
    CK(tt_geometry(&T, tmeas, trec, tcent, st));
    CK(tt_geometry(&S, smeas, srec, scent, st));
    T.measure = tmeas;   /* generated meshes are CCW: the signed measure is |measure| */
    S.measure = smeas;

    /* source grid: nx = ny = int(sqrt(E)) over the bbox (locate.py:38-41) */
    tt_grid_t G = {0};
    G.dim = 2;
    G.n[0] = G.n[1] = (int)sqrt((double)sne);
    G.n[2] = 1;
    G.lo[0] = G.lo[1] = 0.0;
    G.hi[0] = G.hi[1] = 1.0;
    G.n_elems = sne;
    G.rec = srec;
    G.centroids = scent;
    const int64_t ncell = (int64_t)G.n[0] * G.n[1];
    int64_t *cstart, *cursor, total = 0;
    CU(cudaMalloc((void**)&cstart, 8 * (ncell + 1)));
    CU(cudaMalloc((void**)&cursor, 8 * ncell));
    G.cell_start = cstart;
    CK(tt_grid_count(&S, &G, cstart, st));
    CU(cudaMemcpy(&total, cstart + ncell, 8, cudaMemcpyDeviceToHost));
    int32_t* celems;
    CU(cudaMalloc((void**)&celems, 4 * total));
    CK(tt_grid_fill(&S, &G, celems, cursor, st));
    G.cell_elems = celems;

    /* node incidence (target: load reduction + mass; source: walk neighbours) */
    int64_t *t_inc_s, *s_inc_s, *cur2;
    int32_t *t_inc, *s_inc;
    CU(cudaMalloc((void**)&t_inc_s, 8 * (tnn + 1))); CU(cudaMalloc((void**)&t_inc, 12 * tne + 16));
    CU(cudaMalloc((void**)&s_inc_s, 8 * (snn + 1))); CU(cudaMalloc((void**)&s_inc, 12 * sne));
    CU(cudaMalloc((void**)&cur2, 8 * (tnn > snn ? tnn : snn)));
    CK(tt_incidence_count(&T, t_inc_s, st)); CK(tt_incidence_fill(&T, t_inc_s, t_inc, cur2, st));
    CK(tt_incidence_count(&S, s_inc_s, st)); CK(tt_incidence_fill(&S, s_inc_s, s_inc, cur2, st));

    /* certified walk: neighbours + margins, compact float records, per-target seeds */
    int32_t* status;
    CU(cudaMalloc((void**)&status, 4));
    CU(cudaMemset(status, 0, 4));
    double* wrec;
    CU(cudaMalloc((void**)&wrec, 8 * TT_WREC_STRIDE(2) * sne));
    CK(tt_grid_walk_prep(&S, s_inc_s, s_inc, 1e-12, srec, wrec, status, st));
    G.walk = 1;
    G.wrec = wrec;
    int32_t* seeds;
    CU(cudaMalloc((void**)&seeds, sizeof(int32_t) * TT_SEED_ANCHORS * tne));
    CK(tt_seed_elements(&G, &T, 0, tne, seeds, NULL, st));

    /* plan: Sobol(N, skip 0) -> barycentric (SamplePlan.build(N, "sobol", 0)) */
    double *par, *lam;
    CU(cudaMalloc((void**)&par, 16 * N));
    CU(cudaMalloc((void**)&lam, 24 * N));
    CK(tt_plan_sobol(2, N, 0, par, st));
    CK(tt_bary_map(2, N, par, lam, st));
    tt_plan_t P = {TT_PLAN_SHARED, 2, N, lam, 0};

    /* source field: nodal interpolant of sin(x)cos(y) + 2 */
    double* c = malloc(8 * snn);
    for (int64_t i = 0; i < snn; ++i) c[i] = sin(sn[2 * i]) * cos(sn[2 * i + 1]) + 2.0;
    double* dc = dup(c, 8 * snn);
    double* grad;
    CU(cudaMalloc((void**)&grad, 32 * sne));
    CK(tt_pack_grad(&S, dc, grad, st));
    tt_source_t src = {0};
    src.kind = TT_SRC_MESH;
    src.outside = TT_OUTSIDE_SNAP;
    src.dim = 2;
    src.grid = G;
    src.src_elems = S.elems;
    src.coeffs = dc;
    src.seeds = seeds;
    src.elem_grad = grad;

    /* fused load + deterministic node reduction (montecarlo.py:110-147) */
    double *contrib, *b;
    CU(cudaMalloc((void**)&contrib, 24 * tne));
    CU(cudaMalloc((void**)&b, 8 * tnn));
    CK(tt_mc_load(&T, 0, tne, &P, &src, contrib, NULL, status, st));
    CK(tt_reduce_nodes(tnn, 3, t_inc_s, t_inc, 0, tne, contrib, b, st));

    /* mass matrix (degree-2 rule local matrix) and PCG (fem.py:78-152) */
    int64_t* rp;
    CU(cudaMalloc((void**)&rp, 8 * (tnn + 1)));
    CK(tt_mass_pattern(&T, t_inc_s, t_inc, rp, status, st));
    int64_t nnz = 0;
    CU(cudaMemcpy(&nnz, rp + tnn, 8, cudaMemcpyDeviceToHost));
    int32_t* ci;
    double* va;
    CU(cudaMalloc((void**)&ci, 4 * nnz));
    CU(cudaMalloc((void**)&va, 8 * nnz));
    const double pts[3][3] = {{2.0 / 3, 1.0 / 6, 1.0 / 6}, {1.0 / 6, 2.0 / 3, 1.0 / 6}, {1.0 / 6, 1.0 / 6, 2.0 / 3}};
    double local[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int q = 0; q < 3; ++q) s += (1.0 / 3) * pts[q][i] * pts[q][j];
            local[3 * i + j] = s;
        }
    CK(tt_mass_fill(&T, t_inc_s, t_inc, local, rp, ci, va, st));
    double *x, *bx, *work;
    tt_pcg_result_t* res;
    CU(cudaMalloc((void**)&x, 8 * tnn));
    CU(cudaMalloc((void**)&bx, 8 * tnn));
    CU(cudaMalloc((void**)&work, 8 * tt_pcg_workspace_doubles(tnn)));
    CU(cudaMalloc((void**)&res, sizeof(tt_pcg_result_t)));
    CK(tt_pcg(tnn, rp, ci, va, b, 1e-14, 10 * tnn, x, bx, work, res, st));

    /* results */
    tt_pcg_result_t r;
    int32_t flags = 0;
    double integral = 0.0, *hx = malloc(8 * tnn), *dint;
    CU(cudaMemcpy(&r, res, sizeof r, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&flags, status, 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(hx, x, 8 * tnn, cudaMemcpyDeviceToHost));
    CU(cudaMalloc((void**)&dint, 8));
    CK(tt_integrate_p1(&T, x, dint, st));
    CU(cudaMemcpy(&integral, dint, 8, cudaMemcpyDeviceToHost));
    double checksum = 0.0;
    for (int64_t i = 0; i < tnn; ++i) checksum += hx[i] * (double)((i % 7) + 1);
    printf("{\"integral\": %.17g, \"iterations\": %lld, \"converged\": %d, \"flags\": %d, "
           "\"checksum\": %.17g, \"n_nodes\": %lld, \"x0\": %.17g}\n",
           integral, (long long)r.iterations, r.converged, flags, checksum, (long long)tnn, hx[0]);
    return (r.converged && !flags) ? 0 : 2;
}
