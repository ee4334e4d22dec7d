// k_state.cu -- per-group state kernels: fold (slot table -> canonical state,
// the merge of all block partials), Eq. 1 read-out, serialisation, state
// merge and the multi-GPU window exchange.
//
// Canonical device state of a group (int form of the paper's <S, C>,
// PAPER.md:842-853): top lattice index k (int32) and, per level l = 0..K-1
// (absolute level k - l), C_l = floor(T_l / 2^(m-2)) and
// D_l = T_l mod 2^(m-2), i.e. S_l = 1.5 * 2^(W(k-l)) + D_l * u_l.
#include "common.cuh"
#include "internal.h"

namespace repro {

namespace {

constexpr int TPB_STATE = 256;

template <int K>
__device__ __forceinline__ void realign(__int128 (&T)[K], int sh) {
    // the paper's level demotion by `sh` levels
    if (sh <= 0) return;
#pragma unroll
    for (int l = K - 1; l >= 0; --l) T[l] = (l - sh >= 0) ? T[l - sh] : (__int128)0;
}

template <int DT, int K>
__device__ __forceinline__ void load_state(int g, const int64_t *C, const int64_t *D, __int128 (&T)[K]) {
#pragma unroll
    for (int l = 0; l < K; ++l) T[l] = join_CD<DT>(C[(size_t)g * K + l], D[(size_t)g * K + l]);
}

template <int DT, int K>
__device__ __forceinline__ void store_state(int g, const __int128 (&T)[K], int64_t *C, int64_t *D,
                                            int64_t (&Cc)[K], int64_t (&Dc)[K]) {
#pragma unroll
    for (int l = 0; l < K; ++l) {
        split_CD<DT>(T[l], Cc[l], Dc[l]);
        if (C) {
            C[(size_t)g * K + l] = Cc[l];
            D[(size_t)g * K + l] = Dc[l];
        }
    }
}

__device__ __forceinline__ void publish_flags(uint32_t flags, uint32_t *status) {
    flags = __reduce_or_sync(__activemask(), flags);
    if (flags && (threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicOr(status, flags);
}

// slots + kglob -> canonical state (optionally merged into acc), optionally Eq. 1
template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_fold(int32_t G, const int32_t *__restrict__ kglob, const unsigned long long *__restrict__ slots, int merge,
       int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, typename Fmt<DT>::V *out, uint32_t *status) {
    constexpr int NS = Fmt<DT>::KMAX + K;
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= G) return;
    uint32_t flags = 0;
    int k = kglob[g];
    __int128 T[K];
#pragma unroll
    for (int l = 0; l < K; ++l) {
        const unsigned long long *p = slots + ((size_t)g * NS + (k - l + K - 1)) * 2;
        T[l] = ((__int128)(long long)p[1] << 32) + (__int128)p[0];
    }
    if (merge) {
        const int ka = acc_k[g];
        __int128 Ta[K];
        load_state<DT, K>(g, acc_C, acc_D, Ta);
        const int kn = max(k, ka);
        realign<K>(T, kn - k);
        realign<K>(Ta, kn - ka);
#pragma unroll
        for (int l = 0; l < K; ++l) T[l] += Ta[l];
        k = kn;
    }
    int64_t Cc[K], Dc[K];
    store_state<DT, K>(g, T, acc_k ? acc_C : nullptr, acc_D, Cc, Dc);
    if (acc_k) acc_k[g] = k;
    if (out) out[g] = eq1_finalize<DT, K>(k, Cc, Dc, flags);
    publish_flags(flags, status);
}

template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_finalize(int32_t G, const int32_t *__restrict__ k, const int64_t *__restrict__ C,
           const int64_t *__restrict__ D, typename Fmt<DT>::V *out, uint32_t *status) {
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= G) return;
    uint32_t flags = 0;
    int64_t Cc[K], Dc[K];
#pragma unroll
    for (int l = 0; l < K; ++l) { Cc[l] = C[(size_t)g * K + l]; Dc[l] = D[(size_t)g * K + l]; }
    out[g] = eq1_finalize<DT, K>(k[g], Cc, Dc, flags);
    publish_flags(flags, status);
}

// SPEC.md:277 layout: per group S[0..K) then C[0..K) in the value type.
template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_export(int32_t G, const int32_t *__restrict__ k, const int64_t *__restrict__ C,
         const int64_t *__restrict__ D, typename Fmt<DT>::V *state, uint32_t *status) {
    using F = Fmt<DT>;
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= G) return;
    uint32_t flags = 0;
#pragma unroll
    for (int l = 0; l < K; ++l) {
        const int e = F::W * (k[g] - l);
        const int64_t c = C[(size_t)g * K + l], d = D[(size_t)g * K + l];
        const typename F::V S = F::add(F::mul(F::from_i64(3), F::pow2(e - 1)),
                                       F::mul(F::from_i64(d), F::pow2(e - F::m)));
        if ((double)(c < 0 ? -c : c) >= F::CMAX) flags |= FLAG_ERANGE;
        state[(size_t)g * 2 * K + l] = S;
        state[(size_t)g * 2 * K + K + l] = F::from_i64(c);
    }
    publish_flags(flags, status);
}

template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_import(int32_t G, const typename Fmt<DT>::V *__restrict__ state, int32_t *k, int64_t *C, int64_t *D,
         uint32_t *status) {
    using F = Fmt<DT>;
    using Bits = typename F::Bits;
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= G) return;
    uint32_t flags = 0;
    const Bits b0 = F::bits(state[(size_t)g * 2 * K]);
    const int e0 = (int)((b0 >> F::m) & F::EXPMASK) - F::BIAS;
    int kk = e0 / F::W;
    if (e0 < 0 || e0 % F::W != 0 || kk > F::KMAX) { flags |= FLAG_EINVAL; kk = 0; }
#pragma unroll
    for (int l = 0; l < K; ++l) {
        const Bits b = F::bits(state[(size_t)g * 2 * K + l]);
        const int e = (int)((b >> F::m) & F::EXPMASK) - F::BIAS;
        const Bits frac = b & (((Bits)1 << F::m) - 1);
        const Bits sign = b >> (8 * sizeof(Bits) - 1);
        // S_l = 1.5 * 2^e + D u with D < 2^(m-2): fraction bits 10xxx...
        if (sign || e != F::W * (kk - l) || (frac >> (F::m - 2)) != 2) flags |= FLAG_EINVAL;
        const typename F::V c = state[(size_t)g * 2 * K + K + l];
        const double cd = (double)c;
        if (!(cd == trunc(cd)) || fabs(cd) >= F::CMAX) flags |= FLAG_EINVAL;
        D[(size_t)g * K + l] = (int64_t)(frac & (((Bits)1 << (F::m - 2)) - 1));
        C[(size_t)g * K + l] = (int64_t)cd;
    }
    k[g] = kk;
    publish_flags(flags, status);
}

template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_merge_state(int32_t G, int32_t *dk, int64_t *dC, int64_t *dD, const int32_t *sk, const int64_t *sC,
              const int64_t *sD) {  // src may alias dst (dst += dst): each thread reads its group before writing
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= G) return;
    __int128 Ta[K], Tb[K];
    load_state<DT, K>(g, dC, dD, Ta);
    load_state<DT, K>(g, sC, sD, Tb);
    const int ka = dk[g], kb = sk[g], kn = max(ka, kb);
    realign<K>(Ta, kn - ka);
    realign<K>(Tb, kn - kb);
#pragma unroll
    for (int l = 0; l < K; ++l) Ta[l] += Tb[l];
    int64_t Cc[K], Dc[K];
    store_state<DT, K>(g, Ta, dC, dD, Cc, Dc);
    dk[g] = kn;
}

// realigned level sums as carry-split limbs (lo in [0, 2^32), hi = T >> 32)
template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_window_export(int32_t G, const int32_t *__restrict__ k, const int64_t *__restrict__ C,
                const int64_t *__restrict__ D, const int32_t *__restrict__ kg, int64_t *limbs,
                uint32_t *status) {
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= G) return;
    uint32_t flags = 0;
    __int128 T[K];
    load_state<DT, K>(g, C, D, T);
    const int sh = kg[g] - k[g];
    if (sh < 0) flags |= FLAG_EINVAL;
    realign<K>(T, sh);
#pragma unroll
    for (int l = 0; l < K; ++l) {
        limbs[((size_t)g * K + l) * 2 + 0] = (int64_t)(T[l] & 0xFFFFFFFF);
        limbs[((size_t)g * K + l) * 2 + 1] = (int64_t)(T[l] >> 32);
    }
    publish_flags(flags, status);
}

template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_window_import(int32_t count, const int32_t *__restrict__ kg, const int64_t *__restrict__ limbs,
                int32_t *k, int64_t *C, int64_t *D) {
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= count) return;
    __int128 T[K];
#pragma unroll
    for (int l = 0; l < K; ++l)
        T[l] = ((__int128)limbs[((size_t)g * K + l) * 2 + 1] << 32) + (__int128)limbs[((size_t)g * K + l) * 2 + 0];
    int64_t Cc[K], Dc[K];
    store_state<DT, K>(g, T, C, D, Cc, Dc);
    k[g] = kg[g];
}

// Multi-GPU exchange of the absolute-level slot table: the
// K slot words under each group's GLOBAL top (the realignment of the paper's
// demotion, is just a choice of slots), as int64 pairs
// [g][l][lo, hi] for an integer SUM across ranks.
template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_slot_limbs(int32_t G, const int32_t *__restrict__ kg, const unsigned long long *__restrict__ slots,
             int64_t *__restrict__ limbs) {
    constexpr int NS = Fmt<DT>::KMAX + K;
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= G) return;
    const int k = kg[g];
#pragma unroll
    for (int l = 0; l < K; ++l) {
        const unsigned long long *p = slots + ((size_t)g * NS + (k - l + K - 1)) * 2;
        limbs[((size_t)g * K + l) * 2] = (int64_t)p[0];
        limbs[((size_t)g * K + l) * 2 + 1] = (int64_t)p[1];
    }
}

// canonical state + Eq. 1 of `count` groups from summed limbs (kg, limbs and
// out indexed from the range's first group)
template <int DT, int K>
__global__ void __launch_bounds__(TPB_STATE)
k_limbs_finalize(int32_t count, const int32_t *__restrict__ kg, const int64_t *__restrict__ limbs,
                 typename Fmt<DT>::V *out, uint32_t *status) {
    const int g = blockIdx.x * TPB_STATE + threadIdx.x;
    if (g >= count) return;
    uint32_t flags = 0;
    __int128 T[K];
#pragma unroll
    for (int l = 0; l < K; ++l)
        T[l] = ((__int128)limbs[((size_t)g * K + l) * 2 + 1] << 32) + (__int128)(unsigned long long)limbs[((size_t)g * K + l) * 2];
    int64_t Cc[K], Dc[K];
    store_state<DT, K>(g, T, nullptr, nullptr, Cc, Dc);
    out[g] = eq1_finalize<DT, K>(kg[g], Cc, Dc, flags);
    publish_flags(flags, status);
}

__global__ void k_status(const uint32_t *flags, int32_t *d_status) {
    const uint32_t f = *flags;
    d_status[0] = (f & FLAG_ESTALL) ? -5 : (f & FLAG_EINVAL) ? -1 : (f & FLAG_EKEY) ? -2 : (f & FLAG_EDOM) ? -3 : (f & FLAG_ERANGE) ? -4 : 0;
}

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + TPB_STATE - 1) / TPB_STATE); }

}  // namespace

#define DISPATCH(DT, K, CALL)                                                   \
    do {                                                                        \
        if (DT == 1) {                                                          \
            if (K == 1) { constexpr int dt_ = 1, k_ = 1; CALL; }                \
            else if (K == 2) { constexpr int dt_ = 1, k_ = 2; CALL; }           \
            else if (K == 3) { constexpr int dt_ = 1, k_ = 3; CALL; }           \
            else if (K == 4) { constexpr int dt_ = 1, k_ = 4; CALL; }           \
            else return -1;                                                     \
        } else {                                                                \
            if (K == 1) { constexpr int dt_ = 0, k_ = 1; CALL; }                \
            else if (K == 2) { constexpr int dt_ = 0, k_ = 2; CALL; }           \
            else if (K == 3) { constexpr int dt_ = 0, k_ = 3; CALL; }           \
            else if (K == 4) { constexpr int dt_ = 0, k_ = 4; CALL; }           \
            else return -1;                                                     \
        }                                                                       \
    } while (0)

#define LAUNCH_TAIL()                                   \
    ++*launches;                                        \
    return cudaGetLastError() == cudaSuccess ? 0 : -2

int launch_slot_limbs(int DT, int K, int32_t G, const int32_t *kg, const unsigned long long *slots, int64_t *limbs,
                      cudaStream_t st, int *launches) {
    if (G == 0) return 0;
    DISPATCH(DT, K, (k_slot_limbs<dt_, k_><<<blocks_for(G), TPB_STATE, 0, st>>>(G, kg, slots, limbs)));
    LAUNCH_TAIL();
}

int launch_limbs_finalize(int DT, int K, int32_t count, const int32_t *kg, const int64_t *limbs, void *out,
                          uint32_t *status, cudaStream_t st, int *launches) {
    if (count == 0) return 0;
    DISPATCH(DT, K, (k_limbs_finalize<dt_, k_><<<blocks_for(count), TPB_STATE, 0, st>>>(
                        count, kg, limbs, (typename Fmt<dt_>::V *)out, status)));
    LAUNCH_TAIL();
}

int launch_fold(int DT, int K, int32_t G, const int32_t *kglob, const unsigned long long *slots, int merge,
                int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out, uint32_t *status,
                cudaStream_t st, int *launches) {
    DISPATCH(DT, K, (k_fold<dt_, k_><<<blocks_for(G), TPB_STATE, 0, st>>>(
                        G, kglob, slots, merge, acc_k, acc_C, acc_D, (typename Fmt<dt_>::V *)out, status)));
    LAUNCH_TAIL();
}

int launch_finalize(int DT, int K, int32_t G, const int32_t *k, const int64_t *C, const int64_t *D, void *out,
                    uint32_t *status, cudaStream_t st, int *launches) {
    DISPATCH(DT, K, (k_finalize<dt_, k_><<<blocks_for(G), TPB_STATE, 0, st>>>(
                        G, k, C, D, (typename Fmt<dt_>::V *)out, status)));
    LAUNCH_TAIL();
}

int launch_export(int DT, int K, int32_t G, const int32_t *k, const int64_t *C, const int64_t *D, void *state,
                  uint32_t *status, cudaStream_t st, int *launches) {
    DISPATCH(DT, K, (k_export<dt_, k_><<<blocks_for(G), TPB_STATE, 0, st>>>(
                        G, k, C, D, (typename Fmt<dt_>::V *)state, status)));
    LAUNCH_TAIL();
}

int launch_import(int DT, int K, int32_t G, const void *state, int32_t *k, int64_t *C, int64_t *D,
                  uint32_t *status, cudaStream_t st, int *launches) {
    DISPATCH(DT, K, (k_import<dt_, k_><<<blocks_for(G), TPB_STATE, 0, st>>>(
                        G, (const typename Fmt<dt_>::V *)state, k, C, D, status)));
    LAUNCH_TAIL();
}

int launch_merge_state(int DT, int K, int32_t G, int32_t *dk, int64_t *dC, int64_t *dD, const int32_t *sk,
                       const int64_t *sC, const int64_t *sD, uint32_t *status, cudaStream_t st,
                       int *launches) {
    (void)status;
    DISPATCH(DT, K, (k_merge_state<dt_, k_><<<blocks_for(G), TPB_STATE, 0, st>>>(G, dk, dC, dD, sk, sC, sD)));
    LAUNCH_TAIL();
}

int launch_window_export(int DT, int K, int32_t G, const int32_t *k, const int64_t *C, const int64_t *D,
                         const int32_t *kg, int64_t *limbs, uint32_t *status, cudaStream_t st,
                         int *launches) {
    DISPATCH(DT, K, (k_window_export<dt_, k_><<<blocks_for(G), TPB_STATE, 0, st>>>(G, k, C, D, kg, limbs,
                                                                                   status)));
    LAUNCH_TAIL();
}

int launch_window_import(int DT, int K, int32_t count, const int32_t *kg, const int64_t *limbs, int32_t *k,
                         int64_t *C, int64_t *D, uint32_t *status, cudaStream_t st, int *launches) {
    (void)status;
    DISPATCH(DT, K, (k_window_import<dt_, k_><<<blocks_for(count), TPB_STATE, 0, st>>>(count, kg, limbs, k,
                                                                                       C, D)));
    LAUNCH_TAIL();
}

int launch_reset(int K, int32_t G, int32_t *k, int64_t *C, int64_t *D, cudaStream_t st, int *launches) {
    (void)launches;
    if (cudaMemsetAsync(k, 0, sizeof(int32_t) * (size_t)G, st) != cudaSuccess) return -2;
    if (cudaMemsetAsync(C, 0, sizeof(int64_t) * (size_t)G * K, st) != cudaSuccess) return -2;
    if (cudaMemsetAsync(D, 0, sizeof(int64_t) * (size_t)G * K, st) != cudaSuccess) return -2;
    return 0;
}

int launch_status(const uint32_t *flags, int32_t *d_status, cudaStream_t st, int *launches) {
    k_status<<<1, 1, 0, st>>>(flags, d_status);
    LAUNCH_TAIL();
}

}  // namespace repro
