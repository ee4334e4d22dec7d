// k_multi.cu -- multi-column reproducible GroupBy in one pass over the rows
// (repro_groupby_sum_multi): several SUMs and COUNT
// of one key column, optionally over the row projection of BASELINE config 4
// (reading A-15), as virtual groups of the on-chip kernel.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"
#include "onchip_launch.cuh"

#include <algorithm>

namespace repro {

// Multi-column on-chip GroupBy (repro_groupby_sum_multi): proj 1 = the
// config-4 projection over (qty, price, disc, tax), proj 0 = ncols columns
// summed independently; both add COUNT as the last virtual column.  Virtual
// groups j * G + g; -1 when the shape has no fused kernel (the caller falls
// back to one pass per column).
int multi_virtual_columns(int proj, int ncols) {
    if (proj == 1) return ncols == 4 ? SrcQ1::NV : -1;
    if (proj == 2) return ncols == 1 ? SrcMoments<1>::NV : -1;
    return (ncols == 1 || ncols == 2 || ncols == 4) ? ncols + 1 : -1;
}

int launch_onchip_multi(int DT, int K, int proj, int ncols, const int32_t *keys, const void *const *cols, int64_t n,
                        int32_t G, int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                        int *launches) {
    const int nv = multi_virtual_columns(proj, ncols);
    if (nv < 0 || (int64_t)G * nv > OnchipCfg<1, 1>::REG_GQ) return -1;
    const int32_t Gv = G * nv;
#define MULTI_K(dt, SRCT)                                                                                     \
    do {                                                                                                      \
        SRCT src;                                                                                             \
        for (int j = 0; j < SRCT::NCOL; ++j) src.col[j] = (const typename Fmt<dt>::V *)cols[j];              \
        src.G = G;                                                                                            \
        switch (K) {                                                                                          \
            case 1: return launch_onchip_src<dt, 1, SRCT, false>(keys, src, n, Gv, kglob, slots, status, st, launches); \
            case 2: return launch_onchip_src<dt, 2, SRCT, false>(keys, src, n, Gv, kglob, slots, status, st, launches); \
            case 3: return launch_onchip_src<dt, 3, SRCT, false>(keys, src, n, Gv, kglob, slots, status, st, launches); \
            case 4: return launch_onchip_src<dt, 4, SRCT, false>(keys, src, n, Gv, kglob, slots, status, st, launches); \
        }                                                                                                     \
        return -1;                                                                                            \
    } while (0)
    // a handful of groups (config 4's shape): per-warp lane-copy tables
    // (k_lean.cu); 1 = not handled there
    const int lr = launch_lean_multi(DT, K, proj, ncols, keys, cols, n, G, kglob, slots, status, st, launches);
    if (lr != 1) return lr;
    using C64_1 = SrcCols<1, 1>;
    using C64_2 = SrcCols<1, 2>;
    using C64_4 = SrcCols<1, 4>;
    using C32_1 = SrcCols<0, 1>;
    using C32_2 = SrcCols<0, 2>;
    using C32_4 = SrcCols<0, 4>;
    if (proj == 1) {
        if (DT != 1) return -1;
        MULTI_K(1, SrcQ1);
    }
    if (proj == 2) {
        using M64 = SrcMoments<1>;
        using M32 = SrcMoments<0>;
        if (DT == 1) MULTI_K(1, M64);
        MULTI_K(0, M32);
    }
    if (DT == 1) {
        if (ncols == 1) MULTI_K(1, C64_1);
        if (ncols == 2) MULTI_K(1, C64_2);
        if (ncols == 4) MULTI_K(1, C64_4);
    } else {
        if (ncols == 1) MULTI_K(0, C32_1);
        if (ncols == 2) MULTI_K(0, C32_2);
        if (ncols == 4) MULTI_K(0, C32_4);
    }
#undef MULTI_K
    return -1;
}

// Keyless single-array SUM (y == nullptr) or dot product x . y (f4): one
// group, no key column (SrcArray), counters with one copy per lane.
int launch_onchip_array(int DT, int K, const void *x, const void *y, int64_t n, int32_t *kglob,
                        unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
#define ARRAY_K(dt, NC)                                                                                          \
    do {                                                                                                         \
        SrcArray<dt, NC> src;                                                                                    \
        src.col[0] = (const typename Fmt<dt>::V *)x;                                                             \
        if (NC == 2) src.col[NC - 1] = (const typename Fmt<dt>::V *)y;                                           \
        src.G = 1;                                                                                               \
        switch (K) {                                                                                             \
            case 1: return launch_onchip_src<dt, 1, SrcArray<dt, NC>, false>(nullptr, src, n, 1, kglob, slots, status, st, launches); \
            case 2: return launch_onchip_src<dt, 2, SrcArray<dt, NC>, false>(nullptr, src, n, 1, kglob, slots, status, st, launches); \
            case 3: return launch_onchip_src<dt, 3, SrcArray<dt, NC>, false>(nullptr, src, n, 1, kglob, slots, status, st, launches); \
            case 4: return launch_onchip_src<dt, 4, SrcArray<dt, NC>, false>(nullptr, src, n, 1, kglob, slots, status, st, launches); \
        }                                                                                                        \
        return -1;                                                                                               \
    } while (0)
    if (DT == 1) {
        if (y) ARRAY_K(1, 2);
        ARRAY_K(1, 1);
    }
    if (y) ARRAY_K(0, 2);
    ARRAY_K(0, 1);
#undef ARRAY_K
}

// ---- helpers of the multi-column entry points ------------------------------

struct OutPtrs {
    void *p[8];
};

// virtual results -> the caller's output columns; COUNT read exactly from the
// slot table: the ones column deposits digit 2^(m - W) (1.0 in units of the
// level-1 ulp 2^(W - m)) per row at absolute level 1, so count = T_1 >> (m - W).
template <int DT, int K>
__global__ void k_multi_scatter(const typename Fmt<DT>::V *__restrict__ vout, int32_t G, int nsum, OutPtrs outs,
                                const unsigned long long *__restrict__ slots, int64_t *counts) {
    using F = Fmt<DT>;
    constexpr int NS = F::KMAX + K;
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    for (int c = 0; c < nsum; ++c) reinterpret_cast<typename F::V *>(outs.p[c])[g] = vout[(size_t)c * G + g];
    if (counts) {
        const size_t vg = (size_t)nsum * G + g;
        const unsigned long long *p = slots + (vg * NS + (1 + K - 1)) * 2;
        const __int128 T = ((__int128)(long long)p[1] << 32) + (__int128)p[0];
        counts[g] = (int64_t)(T >> (F::m - F::W));
    }
}

// config-4 projection columns for the per-column fallback (reading A-15)
__global__ void k_q1_project(const double *__restrict__ price, const double *__restrict__ disc,
                             const double *__restrict__ tax, int64_t n, double *__restrict__ dp,
                             double *__restrict__ charge) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = __dmul_rn(price[i], __dsub_rn(1.0, disc[i]));
        dp[i] = d;
        charge[i] = __dmul_rn(d, __dadd_rn(1.0, tax[i]));
    }
}

// COUNT for the fallback: integer atomics (exact, order-free); bad keys are
// reported by the SUM passes
__global__ void k_count_rows(const int32_t *__restrict__ keys, int64_t n, int32_t G,
                             unsigned long long *counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = keys[i];
        if ((uint32_t)k < (uint32_t)G) atomicAdd(&counts[k], 1ull);
    }
}

__global__ void k_flags_or(uint32_t *acc, const uint32_t *f) { *acc |= *f; }

// x (x) x for the per-column fallback of the moments projection
template <typename V>
__global__ void k_square(const V *__restrict__ x, int64_t n, V *__restrict__ sq) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        sq[i] = sizeof(V) == 8 ? (V)__dmul_rn((double)x[i], (double)x[i]) : (V)__fmul_rn((float)x[i], (float)x[i]);
}

// AVG / sample VARIANCE / STDDEV from the reproducible SUM(x), SUM(x^2) and the
// exact COUNT, each operation rounded once in a fixed order (so the outputs
// are as reproducible as the sums):  avg = s / c,  var = max(0, (q - s*s/c) /
// (c - 1)) (0 for c <= 1), stddev = sqrt(var); an empty group gives 0.
template <typename V>
__global__ void k_moments(const V *__restrict__ s, const V *__restrict__ q, const int64_t *__restrict__ cnt, int32_t G,
                          V *avg, V *var, V *sd) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    const int64_t c = cnt[g];
    V a = V(0), v = V(0);
    if (sizeof(V) == 8) {
        const double cd = (double)c;
        if (c > 0) a = (V)__ddiv_rn((double)s[g], cd);
        if (c > 1) {
            const double t = __dsub_rn((double)q[g], __ddiv_rn(__dmul_rn((double)s[g], (double)s[g]), cd));
            v = (V)fmax(0.0, __ddiv_rn(t, __dsub_rn(cd, 1.0)));
        }
        if (avg) avg[g] = a;
        if (var) var[g] = v;
        if (sd) sd[g] = (V)__dsqrt_rn((double)v);
    } else {
        const float cf = __ll2float_rn(c);
        if (c > 0) a = (V)__fdiv_rn((float)s[g], cf);
        if (c > 1) {
            const float t = __fsub_rn((float)q[g], __fdiv_rn(__fmul_rn((float)s[g], (float)s[g]), cf));
            v = (V)fmaxf(0.0f, __fdiv_rn(t, __fsub_rn(cf, 1.0f)));
        }
        if (avg) avg[g] = a;
        if (var) var[g] = v;
        if (sd) sd[g] = (V)__fsqrt_rn((float)v);
    }
}

int launch_square(int DT, const void *x, int64_t n, void *sq, cudaStream_t st, int *launches) {
    if (n == 0) return 0;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * device_props().sms);
    if (DT == 1) k_square<double><<<blocks, 256, 0, st>>>((const double *)x, n, (double *)sq);
    else k_square<float><<<blocks, 256, 0, st>>>((const float *)x, n, (float *)sq);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_moments(int DT, const void *s, const void *q, const int64_t *cnt, int32_t G, void *avg, void *var, void *sd,
                   cudaStream_t st, int *launches) {
    const int blocks = (G + 255) / 256;
    if (DT == 1)
        k_moments<double><<<blocks, 256, 0, st>>>((const double *)s, (const double *)q, cnt, G, (double *)avg,
                                                  (double *)var, (double *)sd);
    else
        k_moments<float><<<blocks, 256, 0, st>>>((const float *)s, (const float *)q, cnt, G, (float *)avg,
                                                 (float *)var, (float *)sd);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_multi_scatter(int DT, int K, const void *vout, int32_t G, int nsum, void *const *outs,
                         const unsigned long long *slots, int64_t *counts, cudaStream_t st, int *launches) {
    OutPtrs o{};
    for (int c = 0; c < nsum && c < 8; ++c) o.p[c] = outs[c];
    const int tpb = 256, blocks = (G + tpb - 1) / tpb;
#define SCATTER_CASE(dt, k)                                                                                  \
    if (DT == dt && K == k)                                                                                  \
        k_multi_scatter<dt, k><<<blocks, tpb, 0, st>>>((const typename Fmt<dt>::V *)vout, G, nsum, o, slots, counts);
    SCATTER_CASE(1, 1) SCATTER_CASE(1, 2) SCATTER_CASE(1, 3) SCATTER_CASE(1, 4)
    SCATTER_CASE(0, 1) SCATTER_CASE(0, 2) SCATTER_CASE(0, 3) SCATTER_CASE(0, 4)
#undef SCATTER_CASE
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_q1_project(const double *price, const double *disc, const double *tax, int64_t n, double *dp,
                      double *charge, cudaStream_t st, int *launches) {
    if (n == 0) return 0;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * device_props().sms);
    k_q1_project<<<blocks, 256, 0, st>>>(price, disc, tax, n, dp, charge);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_count_rows(const int32_t *keys, int64_t n, int32_t G, int64_t *counts, cudaStream_t st, int *launches) {
    if (cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)G, st) != cudaSuccess) return -2;
    if (n == 0) return 0;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * device_props().sms);
    k_count_rows<<<blocks, 256, 0, st>>>(keys, n, G, (unsigned long long *)counts);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_flags_or(uint32_t *acc, const uint32_t *f, cudaStream_t st, int *launches) {
    k_flags_or<<<1, 1, 0, st>>>(acc, f);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace repro
