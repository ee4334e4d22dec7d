// common.cuh -- device-side arithmetic of the reproducible accumulator.
//
// Integer-digit formulation of Algorithm 1, DESIGN.md
// "Integer-digit formulation".  With the readings of DESIGN.md (A-1 ties away
// from zero, A-2 threshold 2^(W-1) ulp(S^(1)), A-3 f = 0):
//   * level j of the W-lattice has ulp u_j = 2^(W*j - m) (extractor
//     S = 1.5 * 2^(W*j));
//   * a value b needs the window top k*(b) = min{k >= 0 : |b| < 2^(W k + W-1-m)}
//     (Alg. 1 lines 3-9);
//   * its contribution to level j is the integer digit d_j = RA(r / u_j)
//     (round half away from zero), r the remainder after the levels above
//     (Alg. 1 lines 10-16);
//   * a group's state is (k_top, T_j = sum of d_j) and the paper's running
//     sum / carry pair is S = 1.5 ufp + (T mod 2^(m-2)) u, C = floor(T / 2^(m-2))
//     (Alg. 1 lines 17-21).
// Integer sums and maxima are associative, which is what lets the GPU merge
// per-thread, per-block and per-GPU partial states in any order.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace repro {

// device status word bits (OR-ed; precedence EKEY > EDOM > ERANGE on read)
// FLAG_ESTALL: a cross-block wait of the routed path (k_route.cu) gave up
// (reported as REPRO_ECUDA; never expected)
enum : uint32_t { FLAG_EKEY = 1u, FLAG_EDOM = 2u, FLAG_ERANGE = 4u, FLAG_EINVAL = 8u, FLAG_ESTALL = 16u };

template <int DT>
struct Fmt;

// binary64: m = 52, W = 40; largest lattice index 25
// (1.5 * 2^(40*26) overflows: reading A-9).
template <>
struct Fmt<1> {
    using V = double;
    using Bits = uint64_t;
    using Digit = int64_t;
    static constexpr int m = 52, W = 40, KMAX = 25, BIAS = 1023, EXPMASK = 0x7FF;
    static constexpr int LIMBS = 2;  // a digit (|d| <= 2^39) is split into 20+20 bits
    static constexpr double CMAX = 9007199254740992.0;  // |C| < 2^53 is exact
    __device__ __forceinline__ static Bits bits(V x) { return (Bits)__double_as_longlong(x); }
    __device__ __forceinline__ static V from_bits(Bits b) { return __longlong_as_double((long long)b); }
    // 2^e for a normal exponent e
    __device__ __forceinline__ static V pow2(int e) { return from_bits((Bits)(int64_t)(e + BIAS) << m); }
    __device__ __forceinline__ static V add(V a, V b) { return __dadd_rn(a, b); }
    __device__ __forceinline__ static V sub(V a, V b) { return __dsub_rn(a, b); }
    __device__ __forceinline__ static V mul(V a, V b) { return __dmul_rn(a, b); }
    __device__ __forceinline__ static V from_i64(int64_t x) { return __ll2double_rn(x); }
};

// binary32: m = 23, W = 18; largest lattice index 7 (1.5 * 2^144 overflows).
template <>
struct Fmt<0> {
    using V = float;
    using Bits = uint32_t;
    using Digit = int32_t;
    static constexpr int m = 23, W = 18, KMAX = 7, BIAS = 127, EXPMASK = 0xFF;
    static constexpr int LIMBS = 1;  // |d| <= 2^17 fits one int32 counter
    static constexpr double CMAX = 16777216.0;  // |C| < 2^24 (reading A-8)
    __device__ __forceinline__ static Bits bits(V x) { return (Bits)__float_as_uint(x); }
    __device__ __forceinline__ static V from_bits(Bits b) { return __uint_as_float(b); }
    __device__ __forceinline__ static V pow2(int e) { return from_bits((Bits)(e + BIAS) << m); }
    __device__ __forceinline__ static V add(V a, V b) { return __fadd_rn(a, b); }
    __device__ __forceinline__ static V sub(V a, V b) { return __fsub_rn(a, b); }
    __device__ __forceinline__ static V mul(V a, V b) { return __fmul_rn(a, b); }
    __device__ __forceinline__ static V from_i64(int64_t x) { return __ll2float_rn(x); }
};

// Window top needed by b: k*(b) = min{k >= 0 : |b| < 2^(W k + W - 1 - m)}.
// |b| in [2^E, 2^(E+1)) needs E + 1 <= W k + W - 1 - m.  Returns -1 and sets
// EDOM for NaN/Inf, -1 and ERANGE beyond the largest lattice index.
template <int DT>
__device__ __forceinline__ int kstar_of(typename Fmt<DT>::V b, uint32_t &flags) {
    using F = Fmt<DT>;
    const int be = (int)((F::bits(b) >> F::m) & F::EXPMASK);
    if (be == F::EXPMASK) { flags |= FLAG_EDOM; return -1; }
    const int t = be - F::BIAS + 2 + F::m - F::W;  // zero / subnormal: t <= 0
    const int k = (be == 0 || t <= 0) ? 0 : (t + F::W - 1) / F::W;
    if (k > F::KMAX) { flags |= FLAG_ERANGE; return -1; }
    return k;
}

// Digits of b at absolute levels kt, kt-1, ..., kt-K+1 (requires kt >= k*(b)).
// Each level is the paper's extraction step q = (r (+) S) (-) S (Alg. 1 line 11)
// written in units of that level's ulp, where the extractor is M = 1.5 * 2^m
// (ulp(M) = 1): x = r / u with its lowest significand bit forced to 1
// (reading A-1, exact RNE of x == round-half-away of r / u because
// ulp(x) <= 2^(W-1-m) <= 1/4), t = x (+) M, d = t (-) M, read from the bits.
// The remainder r - d u goes to the next level scaled by 2^W (exact).
template <int DT, int K>
__device__ __forceinline__ void digits_of(typename Fmt<DT>::V b, int kt,
                                          typename Fmt<DT>::Digit (&d)[K]) {
    using F = Fmt<DT>;
    using V = typename F::V;
    const V M = F::pow2(F::m) + F::pow2(F::m - 1);  // 1.5 * 2^m
    const typename F::Bits Mb = F::bits(M);
    V s = F::mul(b, F::pow2(F::m - F::W * kt));   // r / u_kt, exact
#pragma unroll
    for (int l = 0; l < K; ++l) {
        const V x = F::from_bits(F::bits(s) | (typename F::Bits)1);
        const V t = F::add(x, M);
        d[l] = (typename F::Digit)(F::bits(t) - Mb);
        if (l + 1 < K) s = F::mul(F::sub(s, F::sub(t, M)), F::pow2(F::W));
    }
}

// ---- canonical state helpers (int128 level sums) --------------------------

// Canonical carry split of a level sum: T = C * 2^(m-2) + D, D in [0, 2^(m-2)).
template <int DT>
__device__ __forceinline__ void split_CD(__int128 T, int64_t &C, int64_t &D) {
    constexpr int s = Fmt<DT>::m - 2;
    D = (int64_t)(T & (((__int128)1 << s) - 1));
    C = (int64_t)(T >> s);
}

template <int DT>
__device__ __forceinline__ __int128 join_CD(int64_t C, int64_t D) {
    return ((__int128)C << (Fmt<DT>::m - 2)) + (__int128)D;
}

// Eq. 1, reverse level order:
//   t_l = (S_l (-) 1.5 ufp(S_l)) (+) 0.25 ufp(S_l) C_l,  Q = t_K (+) ... (+) t_1
// with S_l (-) 1.5 ufp = D_l u_l exactly.  Sets ERANGE if C_l is not exactly
// representable in the value type (reading A-8).
template <int DT, int K>
__device__ __forceinline__ typename Fmt<DT>::V eq1_finalize(int k, const int64_t (&C)[K],
                                                            const int64_t (&D)[K], uint32_t &flags) {
    using F = Fmt<DT>;
    using V = typename F::V;
    V q = V(0);
#pragma unroll
    for (int l = K - 1; l >= 0; --l) {
        const int e = F::W * (k - l);
        if ((double)(C[l] < 0 ? -C[l] : C[l]) >= F::CMAX) flags |= FLAG_ERANGE;
        const V dev = F::mul(F::from_i64(D[l]), F::pow2(e - F::m));  // D u, exact
        const V car = F::mul(F::from_i64(C[l]), F::pow2(e - 2));     // 0.25 ufp C, exact or inf
        const V t = F::add(dev, car);
        q = (l == K - 1) ? t : F::add(q, t);
    }
    return q;
}

}  // namespace repro
