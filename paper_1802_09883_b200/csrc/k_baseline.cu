// k_baseline.cu -- the NON-reproducible GroupBy-SUM the north star compares
// against: plain atomicAdd in the value type (BASELINE.json; the paper's
// "built-in float" aggregation).  Same row loader as the
// reproducible path.  Its result depends on the order in which the atomics
// land.
#include "common.cuh"
#include "internal.h"

namespace repro {

namespace {

constexpr int TPB_BASE = 256;
constexpr int R_BASE = 8;

// variant 0: one global atomicAdd per row (REDG.E.ADD.F64.RN / REDG.E.ADD.F32.FTZ.RN)
template <typename V, typename A>
__global__ void __launch_bounds__(TPB_BASE)
k_base_global(const int32_t *__restrict__ keys, const V *__restrict__ vals, int64_t n, int32_t G, A *out) {
    const int64_t stride = (int64_t)gridDim.x * TPB_BASE * R_BASE;
    for (int64_t base = (int64_t)blockIdx.x * TPB_BASE * R_BASE; base < n; base += stride) {
        int32_t key[R_BASE];
        V val[R_BASE];
#pragma unroll
        for (int i = 0; i < R_BASE; ++i) {
            const int64_t r = base + (int64_t)i * TPB_BASE + threadIdx.x;
            key[i] = r < n ? __ldg(keys + r) : -1;
            val[i] = r < n ? __ldg(vals + r) : V(0);
        }
#pragma unroll
        for (int i = 0; i < R_BASE; ++i)
            if ((uint32_t)key[i] < (uint32_t)G) atomicAdd(out + key[i], (A)val[i]);
    }
}

// variant 1: shared-memory privatised table per block (fp64 / fp32 shared
// atomicAdd are CAS loops on sm_100a), flushed with global atomics
template <typename V, typename A>
__global__ void __launch_bounds__(TPB_BASE)
k_base_smem(const int32_t *__restrict__ keys, const V *__restrict__ vals, int64_t n, int32_t G, A *out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    A *tab = reinterpret_cast<A *>(smem_raw);
    for (int g = threadIdx.x; g < G; g += TPB_BASE) tab[g] = A(0);
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * TPB_BASE * R_BASE;
    for (int64_t base = (int64_t)blockIdx.x * TPB_BASE * R_BASE; base < n; base += stride) {
        int32_t key[R_BASE];
        V val[R_BASE];
#pragma unroll
        for (int i = 0; i < R_BASE; ++i) {
            const int64_t r = base + (int64_t)i * TPB_BASE + threadIdx.x;
            key[i] = r < n ? __ldg(keys + r) : -1;
            val[i] = r < n ? __ldg(vals + r) : V(0);
        }
#pragma unroll
        for (int i = 0; i < R_BASE; ++i)
            if ((uint32_t)key[i] < (uint32_t)G) atomicAdd(tab + key[i], (A)val[i]);
    }
    __syncthreads();
    for (int g = threadIdx.x; g < G; g += TPB_BASE)
        if (tab[g] != A(0)) atomicAdd(out + g, tab[g]);
}

// variant 2 (G <= 16): per-thread register partials (one select-add per
// group and row), warp shuffle reduction, one global atomic per group per warp
template <typename V, typename A>
__global__ void __launch_bounds__(TPB_BASE)
k_base_regs(const int32_t *__restrict__ keys, const V *__restrict__ vals, int64_t n, int32_t G, A *out) {
    constexpr int GT = 16;
    A acc[GT];
#pragma unroll
    for (int g = 0; g < GT; ++g) acc[g] = A(0);
    const int64_t stride = (int64_t)gridDim.x * TPB_BASE * R_BASE;
    for (int64_t base = (int64_t)blockIdx.x * TPB_BASE * R_BASE; base < n; base += stride) {
        int32_t key[R_BASE];
        V val[R_BASE];
#pragma unroll
        for (int i = 0; i < R_BASE; ++i) {
            const int64_t r = base + (int64_t)i * TPB_BASE + threadIdx.x;
            key[i] = r < n ? __ldg(keys + r) : -1;
            val[i] = r < n ? __ldg(vals + r) : V(0);
        }
#pragma unroll
        for (int i = 0; i < R_BASE; ++i)
#pragma unroll
            for (int g = 0; g < GT; ++g) acc[g] += key[i] == g ? (A)val[i] : A(0);
    }
#pragma unroll
    for (int g = 0; g < GT; ++g) {
        A v = acc[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && g < G && v != A(0)) atomicAdd(out + g, v);
    }
}

// variant 3: warp aggregation -- lanes holding the same key (MATCH.ANY) sum
// their values through shared memory and the lowest one issues the global
// atomic (one atomic per distinct key per warp: skewed keys stop contending)
template <typename V, typename A>
__global__ void __launch_bounds__(TPB_BASE)
k_base_match(const int32_t *__restrict__ keys, const V *__restrict__ vals, int64_t n, int32_t G, A *out) {
    __shared__ A sv[TPB_BASE];
    const int lane = threadIdx.x & 31;
    A *wv = sv + (threadIdx.x & ~31);
    const int64_t stride = (int64_t)gridDim.x * TPB_BASE * R_BASE;
    for (int64_t base = (int64_t)blockIdx.x * TPB_BASE * R_BASE; base < n; base += stride) {
        int32_t key[R_BASE];
        V val[R_BASE];
#pragma unroll
        for (int i = 0; i < R_BASE; ++i) {
            const int64_t r = base + (int64_t)i * TPB_BASE + threadIdx.x;
            key[i] = r < n ? __ldg(keys + r) : -1;
            val[i] = r < n ? __ldg(vals + r) : V(0);
        }
#pragma unroll
        for (int i = 0; i < R_BASE; ++i) {
            const unsigned peers = __match_any_sync(0xffffffffu, key[i]);
            wv[lane] = (A)val[i];
            __syncwarp();
            if (lane == __ffs(peers) - 1 && (uint32_t)key[i] < (uint32_t)G) {
                A s = A(0);
                for (unsigned p = peers; p; p &= p - 1) s += wv[__ffs(p) - 1];
                atomicAdd(out + key[i], s);
            }
            __syncwarp();
        }
    }
}

template <typename V, typename A>
int run(int variant, const int32_t *keys, const void *vals, int64_t n, int32_t G, void *out, cudaStream_t st,
        int *launches) {
    if (cudaMemsetAsync(out, 0, sizeof(A) * (size_t)G, st) != cudaSuccess) return -2;
    if (n == 0) return 0;
    const int sms = device_props().sms;
    int64_t want = (n + TPB_BASE * R_BASE - 1) / (TPB_BASE * R_BASE);
    if (variant == 0 || variant == 2 || variant == 3) {
        if (variant == 2 && G > 16) return -1;
        auto kern = variant == 0 ? k_base_global<V, A> : variant == 2 ? k_base_regs<V, A> : k_base_match<V, A>;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TPB_BASE, 0);
        const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * sms);
        kern<<<(unsigned)grid, TPB_BASE, 0, st>>>(keys, (const V *)vals, n, G, (A *)out);
    } else {
        const size_t smem = sizeof(A) * (size_t)G;
        if (smem > (size_t)device_props().smem_optin) return -1;
        cudaFuncSetAttribute(k_base_smem<V, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_base_smem<V, A>, TPB_BASE, smem);
        if (per_sm < 1) return -1;
        const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * sms);
        k_base_smem<V, A><<<(unsigned)grid, TPB_BASE, smem, st>>>(keys, (const V *)vals, n, G, (A *)out);
    }
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace

int launch_baseline(int DT, int variant, int acc64, const int32_t *keys, const void *vals, int64_t n,
                    int32_t G, void *out, cudaStream_t st, int *launches) {
    if (variant < 0 || variant > 3) return -1;
    if (DT == 1) return run<double, double>(variant, keys, vals, n, G, out, st, launches);
    if (acc64) return run<float, double>(variant, keys, vals, n, G, out, st, launches);
    return run<float, float>(variant, keys, vals, n, G, out, st, launches);
}

}  // namespace repro
