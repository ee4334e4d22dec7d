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
// group and row), warp shuffle reduction, one global atomic per group per
// warp.  Rows stream in 16-byte vectors (4 rows per load of keys), R_BASE / 4
// quads per thread in flight; a ragged or unaligned remainder is scalar.
template <typename V, typename A>
__global__ void __launch_bounds__(TPB_BASE)
k_base_regs(const int32_t *__restrict__ keys, const V *__restrict__ vals, int64_t n, int32_t G, A *out) {
    constexpr int GT = 16, QB = R_BASE / 4;
    A acc[GT];
#pragma unroll
    for (int g = 0; g < GT; ++g) acc[g] = A(0);
    auto add = [&](int32_t k, V v) {
#pragma unroll
        for (int g = 0; g < GT; ++g) acc[g] += k == g ? (A)v : A(0);
    };
    const bool vec = ((((uintptr_t)keys) | ((uintptr_t)vals)) & 15) == 0;
    const int64_t nq = vec ? n / 4 : 0;
    const int64_t stride = (int64_t)gridDim.x * TPB_BASE * QB;
    for (int64_t base = (int64_t)blockIdx.x * TPB_BASE * QB; base < nq; base += stride) {
        int4 kk[QB];
        V vv[QB][4];
#pragma unroll
        for (int i = 0; i < QB; ++i) {
            const int64_t q = base + (int64_t)i * TPB_BASE + threadIdx.x;
            if (q < nq) {
                kk[i] = __ldcs(reinterpret_cast<const int4 *>(keys) + q);
                if constexpr (sizeof(V) == 8) {
                    const double2 a = __ldcs(reinterpret_cast<const double2 *>(vals) + 2 * q);
                    const double2 b = __ldcs(reinterpret_cast<const double2 *>(vals) + 2 * q + 1);
                    vv[i][0] = a.x; vv[i][1] = a.y; vv[i][2] = b.x; vv[i][3] = b.y;
                } else {
                    const float4 a = __ldcs(reinterpret_cast<const float4 *>(vals) + q);
                    vv[i][0] = a.x; vv[i][1] = a.y; vv[i][2] = a.z; vv[i][3] = a.w;
                }
            } else {
                kk[i] = make_int4(-1, -1, -1, -1);
#pragma unroll
                for (int u = 0; u < 4; ++u) vv[i][u] = V(0);
            }
        }
#pragma unroll
        for (int i = 0; i < QB; ++i) {
            add(kk[i].x, vv[i][0]);
            add(kk[i].y, vv[i][1]);
            add(kk[i].z, vv[i][2]);
            add(kk[i].w, vv[i][3]);
        }
    }
    for (int64_t r = 4 * nq + (int64_t)blockIdx.x * TPB_BASE + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB_BASE)
        add(__ldg(keys + r), __ldg(vals + r));
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

// variant 4: heavy hitters privatised.  A sampling kernel picks the keys
// holding >= 1/2048 of 8192 evenly spaced rows (at most HH_MAX); every warp
// sums its rows of those keys in a private shared-memory table (equal keys of
// a warp are first combined through MATCH.ANY; the leader adds without an
// atomic: the table is the warp's), the other rows go to global atomicAdd, and
// each block flushes its heavy sums with one global atomic per key.  Skewed
// keys (Zipf's head) stop serialising on a few global addresses.
constexpr int HH_MAX = 256, HH_SLOTS = 512, HH_SAMPLE = 8192, HH_SHASH = 16384;
__device__ int32_t g_hh_keys[HH_MAX];
__device__ int g_hh_n;

__global__ void __launch_bounds__(1024) k_base_hh_sample(const int32_t *__restrict__ keys, int64_t n, int32_t G) {
    extern __shared__ int2 hs[];  // (key, count), key -1 = empty
    __shared__ int s_n;
    const int tid = threadIdx.x;
    for (int i = tid; i < HH_SHASH; i += 1024) hs[i] = make_int2(-1, 0);
    if (tid == 0) s_n = 0;
    __syncthreads();
    for (int i = tid; i < HH_SAMPLE; i += 1024) {
        const int64_t r = n * i / HH_SAMPLE;
        if (r >= n) continue;
        const int32_t k = keys[r];
        if ((uint32_t)k >= (uint32_t)G) continue;
        uint32_t h = ((uint32_t)k * 0x9E3779B1u) >> 18;
        for (;;) {
            const int old = atomicCAS(&hs[h].x, -1, k);
            if (old == -1 || old == k) { atomicAdd(&hs[h].y, 1); break; }
            h = (h + 1) & (HH_SHASH - 1);
        }
    }
    __syncthreads();
    const int thr = max(2, (int)min((int64_t)HH_SAMPLE, n) / 2048);
    for (int i = tid; i < HH_SHASH; i += 1024)
        if (hs[i].x >= 0 && hs[i].y >= thr) {
            const int s = atomicAdd(&s_n, 1);
            if (s < HH_MAX) g_hh_keys[s] = hs[i].x;
        }
    __syncthreads();
    if (tid == 0) g_hh_n = min(s_n, HH_MAX);
}

template <typename V, typename A>
__global__ void __launch_bounds__(TPB_BASE)
k_base_hh(const int32_t *__restrict__ keys, const V *__restrict__ vals, int64_t n, int32_t G, A *out) {
    constexpr int NW = TPB_BASE / 32;
    __shared__ int2 hmap[HH_SLOTS];             // key -> heavy index
    __shared__ A wacc[NW][HH_MAX];              // per-warp heavy sums
    __shared__ A sv[TPB_BASE];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nh = g_hh_n;
    for (int i = tid; i < HH_SLOTS; i += TPB_BASE) hmap[i] = make_int2(-1, -1);
    for (int i = tid; i < NW * HH_MAX; i += TPB_BASE) (&wacc[0][0])[i] = A(0);
    __syncthreads();
    if (tid == 0)
        for (int h = 0; h < nh; ++h) {
            const int32_t k = g_hh_keys[h];
            uint32_t s_ = ((uint32_t)k * 0x9E3779B1u) >> 23;
            while (hmap[s_].x != -1) s_ = (s_ + 1) & (HH_SLOTS - 1);
            hmap[s_] = make_int2(k, h);
        }
    __syncthreads();
    A *wv = sv + (tid & ~31);
    const int64_t stride = (int64_t)gridDim.x * TPB_BASE * R_BASE;
    for (int64_t base = (int64_t)blockIdx.x * TPB_BASE * R_BASE; base < n; base += stride) {
        int32_t key[R_BASE];
        V val[R_BASE];
#pragma unroll
        for (int i = 0; i < R_BASE; ++i) {
            const int64_t r = base + (int64_t)i * TPB_BASE + tid;
            key[i] = r < n ? __ldg(keys + r) : -1;
            val[i] = r < n ? __ldg(vals + r) : V(0);
        }
#pragma unroll
        for (int i = 0; i < R_BASE; ++i) {
            const bool ok = (uint32_t)key[i] < (uint32_t)G;
            int hidx = -1;
            if (ok && nh) {
                uint32_t s_ = ((uint32_t)key[i] * 0x9E3779B1u) >> 23;
                for (;;) {
                    const int2 e = hmap[s_];
                    if (e.x == key[i]) { hidx = e.y; break; }
                    if (e.x == -1) break;
                    s_ = (s_ + 1) & (HH_SLOTS - 1);
                }
            }
            if (ok && hidx < 0) atomicAdd(out + key[i], (A)val[i]);
            if (__any_sync(0xffffffffu, hidx >= 0)) {
                const unsigned peers = __match_any_sync(0xffffffffu, hidx >= 0 ? hidx : -2 - lane);
                wv[lane] = (A)val[i];
                __syncwarp();
                if (hidx >= 0 && lane == __ffs(peers) - 1) {
                    A s = A(0);
                    for (unsigned p = peers; p; p &= p - 1) s += wv[__ffs(p) - 1];
                    wacc[warp][hidx] += s;
                }
                __syncwarp();
            }
        }
    }
    __syncthreads();
    for (int h = tid; h < nh; h += TPB_BASE) {
        A s = A(0);
#pragma unroll
        for (int w = 0; w < NW; ++w) s += wacc[w][h];
        if (s != A(0)) atomicAdd(out + g_hh_keys[h], s);
    }
}

template <typename V, typename A>
int run(int variant, const int32_t *keys, const void *vals, int64_t n, int32_t G, void *out, cudaStream_t st,
        int *launches) {
    if (cudaMemsetAsync(out, 0, sizeof(A) * (size_t)G, st) != cudaSuccess) return -2;
    if (n == 0) return 0;
    const int sms = device_props().sms;
    int64_t want = (n + TPB_BASE * R_BASE - 1) / (TPB_BASE * R_BASE);
    if (variant == 4) {
        const size_t sm_s = sizeof(int2) * HH_SHASH;
        cudaFuncSetAttribute(k_base_hh_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_s);
        k_base_hh_sample<<<1, 1024, sm_s, st>>>(keys, n, G);
        ++*launches;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_base_hh<V, A>, TPB_BASE, 0);
        const int64_t grid = std::min<int64_t>(want, (int64_t)std::max(per_sm, 1) * sms);
        k_base_hh<V, A><<<(unsigned)grid, TPB_BASE, 0, st>>>(keys, (const V *)vals, n, G, (A *)out);
    } else if (variant == 0 || variant == 2 || variant == 3) {
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
    if (variant < 0 || variant > 4) return -1;
    if (DT == 1) return run<double, double>(variant, keys, vals, n, G, out, st, launches);
    if (acc64) return run<float, double>(variant, keys, vals, n, G, out, st, launches);
    return run<float, float>(variant, keys, vals, n, G, out, st, launches);
}

}  // namespace repro
