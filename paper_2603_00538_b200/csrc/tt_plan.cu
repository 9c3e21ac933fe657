// Sample plans: Sobol (Gray-code, Joe-Kuo dims 1-3), PCG64 (numpy default_rng stream,
// jump-ahead per draw), Philox4x32-10 per-element streams, barycentric maps.
//
// sobol.py:34-52 / montecarlo.py:68-107 are the reference; all integer work is exact and
// the float scalings are exact (2^-32, 2^-53), so plans are bit-identical to numpy for
// d = 2 (sqrt is IEEE correctly rounded on sm_100a).
#include "tt_common.cuh"
#include "tt_philox.cuh"

namespace tt {

struct SobolDirs {
    uint32_t v[3][32];
};

static SobolDirs make_sobol_dirs() {
    SobolDirs s;
    for (int k = 0; k < 32; ++k) s.v[0][k] = 1u << (31 - k);
    uint64_t m2[32], m3[32];
    m2[0] = 1;
    for (int k = 1; k < 32; ++k) m2[k] = (m2[k - 1] << 1) ^ m2[k - 1];        // s=1, a=0
    m3[0] = 1; m3[1] = 3;
    for (int k = 2; k < 32; ++k) m3[k] = (m3[k - 1] << 1) ^ (m3[k - 2] << 2) ^ m3[k - 2];  // s=2, a=1
    for (int k = 0; k < 32; ++k) {
        s.v[1][k] = (uint32_t)(m2[k] << (31 - k));
        s.v[2][k] = (uint32_t)(m3[k] << (31 - k));
    }
    return s;
}

__global__ void sobol_kernel(SobolDirs dirs, int dim, int64_t count, int64_t skip,
                             double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint64_t idx = (uint64_t)(1 + skip + i);
    uint64_t gray = idx ^ (idx >> 1);
    for (int d = 0; d < dim; ++d) {
        uint32_t acc = 0;
        for (int k = 0; k < 32; ++k)
            if ((gray >> k) & 1ull) acc ^= dirs.v[d][k];
        out[i * dim + d] = (double)acc * 2.3283064365386963e-10;  // 2^-32, exact
    }
}

// numpy PCG64 (XSL-RR 128/64): draw m uses the state after m+1 LCG steps.
typedef unsigned __int128 u128;
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 delta, u128 mult, u128 plus) {
    u128 acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= mult;
            acc_plus = acc_plus * mult + plus;
        }
        plus = (mult + 1) * plus;
        mult *= mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

__global__ void pcg64_kernel(int dim, int64_t count, uint64_t s_hi, uint64_t s_lo,
                             uint64_t i_hi, uint64_t i_lo, double* __restrict__ out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t total = count * dim;
    if (t >= total) return;
    const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
    u128 state = ((u128)s_hi << 64) | s_lo;
    u128 inc = ((u128)i_hi << 64) | i_lo;
    u128 st = pcg_advance(state, (u128)(t + 1), mult, inc);
    uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
    unsigned rot = (unsigned)(st >> 122);
    uint64_t x = hi ^ lo;
    uint64_t r = (x >> rot) | (x << ((64 - rot) & 63));
    out[t] = (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

template <int D>
__device__ __forceinline__ void bary_map_one(const double* p, double* lam) {
    if constexpr (D == 2) {
        double r = __dsqrt_rn(p[0]);
        lam[0] = sub(1.0, r);
        lam[1] = mul(r, sub(1.0, p[1]));
        lam[2] = mul(r, p[1]);
    } else {
        double r = cbrt(p[0]);
        double q = __dsqrt_rn(p[1]);
        double rq = mul(r, q);
        lam[0] = sub(1.0, r);
        lam[1] = mul(r, sub(1.0, q));
        lam[2] = mul(rq, sub(1.0, p[2]));
        lam[3] = mul(rq, p[2]);
    }
}

template <int D>
__global__ void bary_map_kernel(int64_t count, const double* __restrict__ param,
                                double* __restrict__ lam) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    double p[D], l[D + 1];
#pragma unroll
    for (int c = 0; c < D; ++c) p[c] = param[i * D + c];
    bary_map_one<D>(p, l);
#pragma unroll
    for (int c = 0; c <= D; ++c) lam[i * (D + 1) + c] = l[c];
}

__global__ void philox_param_kernel(int dim, int64_t e_lo, int64_t n_elems, int64_t n_samples,
                                    uint64_t seed, double* __restrict__ out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_elems * n_samples) return;
    int64_t e = e_lo + t / n_samples;
    int64_t j = t % n_samples;
    double xi[3];
    philox_uniforms(seed, (uint64_t)e, (uint64_t)j, xi);
    for (int c = 0; c < dim; ++c) out[t * dim + c] = xi[c];
}

}  // namespace tt

using namespace tt;

extern "C" int tt_plan_sobol(int dim, int64_t count, int64_t skip, double* param, void* stream) {
    if (dim < 1 || dim > 3 || count < 0 || skip < 0) {
        set_error("tt_plan_sobol: bad dim/count/skip (%d, %lld, %lld)", dim, (long long)count,
                  (long long)skip);
        return TT_ERR_INVALID_PARAMETER;
    }
    if (count == 0) return TT_OK;
    static SobolDirs dirs = make_sobol_dirs();
    sobol_kernel<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(dirs, dim, count, skip,
                                                                       param);
    return launch_check("sobol_kernel");
}

extern "C" int tt_plan_pcg64(int dim, int64_t count, uint64_t state_hi, uint64_t state_lo,
                             uint64_t inc_hi, uint64_t inc_lo, double* param, void* stream) {
    if (dim < 1 || dim > 3 || count < 0) {
        set_error("tt_plan_pcg64: bad dim/count");
        return TT_ERR_INVALID_PARAMETER;
    }
    if (count == 0) return TT_OK;
    pcg64_kernel<<<grid_for(count * dim, 256), 256, 0, as_stream(stream)>>>(
        dim, count, state_hi, state_lo, inc_hi, inc_lo, param);
    return launch_check("pcg64_kernel");
}

extern "C" int tt_bary_map(int dim, int64_t count, const double* param, double* lam,
                           void* stream) {
    if (count == 0) return TT_OK;
    if (dim == 2)
        bary_map_kernel<2><<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(count, param, lam);
    else if (dim == 3)
        bary_map_kernel<3><<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(count, param, lam);
    else {
        set_error("tt_bary_map: dim must be 2 or 3");
        return TT_ERR_INVALID_PARAMETER;
    }
    return launch_check("bary_map_kernel");
}

extern "C" int tt_plan_philox(int dim, int64_t e_lo, int64_t e_hi, int64_t n_samples,
                              uint64_t seed, double* param, void* stream) {
    if (dim < 2 || dim > 3 || e_hi < e_lo || n_samples < 1) {
        set_error("tt_plan_philox: bad arguments");
        return TT_ERR_INVALID_PARAMETER;
    }
    int64_t total = (e_hi - e_lo) * n_samples;
    if (total == 0) return TT_OK;
    philox_param_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
        dim, e_lo, e_hi - e_lo, n_samples, seed, param);
    return launch_check("philox_param_kernel");
}
