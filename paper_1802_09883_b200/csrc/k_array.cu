// k_array.cu -- keyless single-array reproducible SUM / dot product (f4 of
// the RSum setting, one accumulator over a whole array,
// PAPER.md:755-757).
//
// With a single group there is nothing to scatter, so the per-group counter
// tables of the on-chip GroupBy kernel (shared-memory atomics) are replaced
// by per-THREAD state in registers: a window top kt and K int64 level sums
// (integer-digit formulation, common.cuh).  Each element's K digits come from
// the paper's extraction step (Alg. 1 lines 10-16) against
// the fixed extractors 1.5 * 2^m * u_l of the thread's window, read back as
// integers from the bits of t = r (+) E_l (same binade as E_l, so
// bits(t) - bits(E_l) is the digit).  A value needing a higher window
// (k*(b) > kt, Alg. 1 lines 3-9) demotes the thread's level sums (PAPER.md:
// 661-664) -- at most KMAX times per thread.  At the end the block aligns
// its threads to the block's highest window (dropping the levels that fall
// below it, exactly as a later demotion would) and publishes K level sums
// into the absolute-level slot table that launch_fold reads; every step is
// integer addition or maximum, so the result is independent of the grid.
//
// Loads: 16-byte vectors, U per thread in flight, contiguous chunk per block
// (a multiple of the vector width, so every vector is aligned when the
// arrays are); the last block takes the n % VEC scalar tail.
#include "common.cuh"
#include "internal.h"

namespace repro {

namespace {

constexpr int ARR_TPB = 256;

template <int DT>
struct Vec;
template <>
struct Vec<1> {
    using T = double2;
    static constexpr int N = 2;
    __device__ __forceinline__ static void get(const T &v, double (&o)[2]) { o[0] = v.x; o[1] = v.y; }
};
template <>
struct Vec<0> {
    using T = float4;
    static constexpr int N = 4;
    __device__ __forceinline__ static void get(const T &v, float (&o)[4]) {
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
};

// Per-thread reproducible accumulator: window top kt, level sums of absolute
// level kt - l, extractors E_l = 1.5 * 2^m * u_(kt-l).  The level sums are
// kept RAW: R[l] accumulates bits(t) (mod 2^64) and `cnt` counts the
// deposits since the extractors were set, so the true level sum is
// R[l] - cnt * bits(E_l) -- one 64-bit add per digit instead of a subtract
// and an add (the modular wrap cancels: the true sum fits an int64).
template <int DT, int K>
struct ThreadAcc {
    using F = Fmt<DT>;
    using V = typename F::V;
    using B = typename F::Bits;
    int kt = 0;
    uint32_t thr;  // |b| < 2^(W kt + W - 1 - m)  <=>  abs bits (high word) < thr
    uint32_t cnt = 0;
    uint64_t R[K];
    V e[K];

    __device__ __forceinline__ void set_window() {
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const int ue = F::W * (kt - l) - F::m;  // log2 u of level kt - l
            e[l] = F::add(F::pow2(ue + F::m), F::pow2(ue + F::m - 1));
        }
        const int elim = F::W * kt + F::W - 1 - F::m + F::BIAS;  // biased exponent bound
        thr = (uint32_t)elim << (DT == 1 ? 20 : 23);
        cnt = 0;
    }
    __device__ __forceinline__ int64_t level(int l) const {
        return (int64_t)(R[l] - (uint64_t)cnt * (uint64_t)(typename F::Bits)F::bits(e[l]));
    }
    __device__ __forceinline__ ThreadAcc() {
#pragma unroll
        for (int l = 0; l < K; ++l) R[l] = 0;
        set_window();
    }
    // raise the window to k > kt: level sums shift down, the lowest drop out
    // (PAPER.md:661-664); the shifted sums are stored raw for the new window
    __device__ __forceinline__ void raise(int k) {
        int64_t T[K];
#pragma unroll
        for (int l = 0; l < K; ++l) T[l] = level(l);
        const int sh = k - kt;
#pragma unroll
        for (int l = K - 1; l >= 0; --l) {
            int64_t v = 0;
#pragma unroll
            for (int s = 1; s < K; ++s)  // static register indices
                if (s == sh && l - s >= 0) v = T[l - s];
            T[l] = v;
        }
        kt = k;
        set_window();
#pragma unroll
        for (int l = 0; l < K; ++l) R[l] = (uint64_t)T[l];
    }
    // deposit one value with k*(b) <= kt (0 for skipped rows): the digit of
    // level l is bits(t) - bits(E_l), t = (r | lsb) (+) E_l (reading A-1)
    __device__ __forceinline__ void deposit(V r) {
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const V x = F::from_bits(F::bits(r) | (B)1);
            const V t = F::add(x, e[l]);
            R[l] += (uint64_t)F::bits(t);
            if (l + 1 < K) r = F::sub(r, F::sub(t, e[l]));
        }
    }
};

// |b|'s high word (binary64) or bits (binary32) without the sign
template <int DT>
__device__ __forceinline__ uint32_t abs_hi(typename Fmt<DT>::V v) {
    if (DT == 1) return (uint32_t)__double2hiint((double)v) & 0x7FFFFFFFu;
    return __float_as_uint((float)v) & 0x7FFFFFFFu;
}

// k*(b) (Alg. 1 lines 3-9); -1 and a flag for a value that must not deposit
template <int DT>
__device__ __forceinline__ int kstar_flag(typename Fmt<DT>::V v, uint32_t &flags) {
    using F = Fmt<DT>;
    const int be = (int)((F::bits(v) >> F::m) & F::EXPMASK);
    const int t = max(be - F::BIAS + 2 + F::m - F::W, 0);
    const int ks = (t + F::W - 1) / F::W;
    const uint32_t bad = be == F::EXPMASK ? FLAG_EDOM : (ks > F::KMAX ? FLAG_ERANGE : 0u);
    flags |= bad;
    return bad ? -1 : ks;
}

template <int DT, int K, int NC, int U>
__global__ void __launch_bounds__(ARR_TPB)
k_rsum(const typename Fmt<DT>::V *__restrict__ x, const typename Fmt<DT>::V *__restrict__ y, int64_t n,
       int64_t chunk, int32_t *__restrict__ kglob, unsigned long long *__restrict__ slots,
       uint32_t *__restrict__ status) {
    using F = Fmt<DT>;
    using V = typename F::V;
    using VT = typename Vec<DT>::T;
    constexpr int VN = Vec<DT>::N;
    const int64_t row0 = (int64_t)blockIdx.x * chunk;
    const int64_t row1 = min(n, row0 + chunk);
    ThreadAcc<DT, K> acc;
    uint32_t flags = 0;

    // one batch of up to U*VN elements per thread: one magnitude compare
    // per element against the window's bound; a batch holding a larger value,
    // NaN/Inf or an out-of-range value takes the exact per-element check
    // (invalid values are flagged and replaced by 0) and raises the window
    auto take = [&](V (&v)[U * VN]) {
        uint32_t mx = 0;
#pragma unroll
        for (int i = 0; i < U * VN; ++i) mx = max(mx, abs_hi<DT>(v[i]));
        if (mx >= acc.thr) {
            int kmax = 0;
#pragma unroll
            for (int i = 0; i < U * VN; ++i) {
                const int ks = kstar_flag<DT>(v[i], flags);
                if (ks < 0) v[i] = V(0);
                kmax = max(kmax, ks);
            }
            if (kmax > acc.kt) acc.raise(kmax);
        }
#pragma unroll
        for (int i = 0; i < U * VN; ++i) acc.deposit(v[i]);
        acc.cnt += U * VN;
    };

    const VT *xv = reinterpret_cast<const VT *>(x + row0);
    const VT *yv = reinterpret_cast<const VT *>(NC == 2 ? y + row0 : x + row0);
    const int64_t nvec = (row1 - row0) / VN;
    constexpr int STEP = U * ARR_TPB;
    int64_t b = 0;
    for (; b + STEP <= nvec; b += STEP) {
        VT a[U], c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = __ldcs(xv + b + u * ARR_TPB + threadIdx.x);
        if (NC == 2) {
#pragma unroll
            for (int u = 0; u < U; ++u) c[u] = __ldcs(yv + b + u * ARR_TPB + threadIdx.x);
        }
        V v[U * VN];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            V p[VN];
            Vec<DT>::get(a[u], p);
            if (NC == 2) {
                V q[VN];
                Vec<DT>::get(c[u], q);
#pragma unroll
                for (int j = 0; j < VN; ++j) p[j] = F::mul(p[j], q[j]);
            }
#pragma unroll
            for (int j = 0; j < VN; ++j) v[u * VN + j] = p[j];
        }
        take(v);
    }
    // remainder of the chunk: whole vectors then scalars, bounds-checked
    for (int64_t e0 = row0 + b * VN; e0 < row1; e0 += (int64_t)U * VN * ARR_TPB) {
        V v[U * VN];
#pragma unroll
        for (int i = 0; i < U * VN; ++i) {
            const int64_t r = e0 + (int64_t)i * ARR_TPB + threadIdx.x;
            V p = r < row1 ? __ldcs(x + r) : V(0);
            if (NC == 2) p = r < row1 ? F::mul(p, __ldcs(y + r)) : V(0);
            v[i] = p;
        }
        take(v);
    }

    // block merge: align to the block's window top, then sum level by level
    __shared__ int kb_s;
    __shared__ int64_t tsum[ARR_TPB / 32][K];
    __shared__ uint32_t fl_s;
    if (threadIdx.x == 0) {
        kb_s = 0;
        fl_s = 0;
    }
    __syncthreads();
    const int kw = __reduce_max_sync(0xffffffffu, acc.kt);
    if ((threadIdx.x & 31) == 0) atomicMax(&kb_s, kw);
    flags = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && flags) atomicOr(&fl_s, flags);
    __syncthreads();
    const int kb = kb_s;
    if (kb > acc.kt) acc.raise(kb);
#pragma unroll
    for (int l = 0; l < K; ++l) {
        int64_t s = acc.level(l);
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) tsum[threadIdx.x >> 5][l] = s;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        const int l = threadIdx.x;
        int64_t s = 0;
#pragma unroll
        for (int w = 0; w < ARR_TPB / 32; ++w) s += tsum[w][l];
        constexpr int NS = F::KMAX + K;
        if (s != 0) {
            unsigned long long *p = slots + (size_t)(kb - l + K - 1) * 2;  // group 0
            atomicAdd(p, (unsigned long long)(s & 0xFFFFFFFFll));
            atomicAdd(p + 1, (unsigned long long)(s >> 32));
        }
        (void)NS;
        if (l == 0) {
            if (kb > 0) atomicMax(kglob, kb);
            if (fl_s) atomicOr(status, fl_s);
        }
    }
}

template <int DT, int K, int NC>
int launch_rsum_t(const void *x, const void *y, int64_t n, int32_t *kglob, unsigned long long *slots,
                  uint32_t *status, cudaStream_t st, int *launches) {
    if (n == 0) return 0;
    constexpr int U = (NC == 2) ? 4 : 8;
    constexpr int VN = Vec<DT>::N;
    auto kern = k_rsum<DT, K, NC, U>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ARR_TPB, 0);
    if (per_sm < 1) return -1;
    int64_t grid = (int64_t)per_sm * device_props().sms;
    // a block's int64 level sums must not overflow: <= 2^23 elements per block
    const int64_t min_grid = (n + (1ll << 23) - 1) >> 23;
    if (grid < min_grid) grid = min_grid;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = (chunk + VN - 1) / VN * VN;
    if (chunk > (1ll << 23)) chunk = (1ll << 23);
    grid = (n + chunk - 1) / chunk;
    kern<<<(unsigned)grid, ARR_TPB, 0, st>>>((const typename Fmt<DT>::V *)x, (const typename Fmt<DT>::V *)y, n,
                                             chunk, kglob, slots, status);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace

int launch_rsum(int DT, int K, const void *x, const void *y, int64_t n, int32_t *kglob, unsigned long long *slots,
                uint32_t *status, cudaStream_t st, int *launches) {
#define RSUM_K(dt, nc)                                                                              \
    switch (K) {                                                                                    \
        case 1: return launch_rsum_t<dt, 1, nc>(x, y, n, kglob, slots, status, st, launches);       \
        case 2: return launch_rsum_t<dt, 2, nc>(x, y, n, kglob, slots, status, st, launches);       \
        case 3: return launch_rsum_t<dt, 3, nc>(x, y, n, kglob, slots, status, st, launches);       \
        case 4: return launch_rsum_t<dt, 4, nc>(x, y, n, kglob, slots, status, st, launches);       \
    }                                                                                               \
    return -1;
    if (DT == 1) {
        if (y) { RSUM_K(1, 2) }
        RSUM_K(1, 1)
    }
    if (y) { RSUM_K(0, 2) }
    RSUM_K(0, 1)
#undef RSUM_K
}

}  // namespace repro
