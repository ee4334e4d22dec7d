// k_onchip.cu -- on-chip (low-cardinality) accumulate kernel.
//
// Hot path rows a1-a4/a6 of SURVEY.md section 8: stream <key, value> rows,
// compute each row's window top k* and its K integer digits (common.cuh),
// and add the digits into a per-block table of the group states held in
// shared memory (HashAggregation with identity hashing, PAPER.md:867-873,
// 1264).  Alg. 1's level check becomes an integer max:
// per tile of rows, every row raises its group's `ktop_next` (shared atomicMax)
// and, after one barrier, groups whose top moved shift their level sums down
// (the paper's demotion) before any digit of the tile is added.
//
// Digits are added with native 32-bit shared atomics (64-bit shared atomics
// are CAS loops on sm_100a): binary64 digits (|d| <= 2^39) are split into a
// 20-bit unsigned low limb and a signed high limb, binary32 digits fit one
// int32.  (MATCH.ANY costs ~64 cycles per warp on sm_100a and REDUX with a
// divergent mask compiles to a serial loop, so there is no general warp
// aggregation; only an all-lanes-same-group warp reduces first.)  Limb counters are folded into
// int64 level sums before they can overflow (Alg. 1's carry propagation,
// PAPER.md:673-679, deferred as in Alg. 2's NB blocking).
//
// At the end each block adds its int64 level sums into a global table indexed
// by ABSOLUTE lattice level (slot j + K - 1 for level j) with 64-bit global
// reductions, and raises the group's global top with atomicMax.  Because a
// row's digit at level j does not depend on which window it was computed in
// (digits above k* are zero), this table is exact whatever the block
// windows were; the fold kernel reads the K slots under the global top.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cstdlib>

namespace repro {

template <int DT, int K>
struct OnchipCfg {
    static constexpr int TPB = 256;
    static constexpr int R = (DT == 1) ? 15 : 16;  // rows per thread per tile
    static constexpr int TILE = TPB * R;           // 3840 / 4096
    // limb counters accept at most LIMIT rows' worth of digits between folds
    static constexpr int LIMIT = (DT == 1) ? 4095 : 16383;
    static constexpr int LIMBS = Fmt<DT>::LIMBS;
    static constexpr int CW = K * LIMBS;  // 32-bit counters per group (group-major)
    static_assert(TILE <= LIMIT, "tile larger than limb headroom");
};

template <int DT, int K>
size_t onchip_smem_bytes(int G) {
    using C = OnchipCfg<DT, K>;
    return (size_t)G * (8 * K + 4 * C::CW + 8);
}

// binary64 digit (|d| <= 2^39) -> 20-bit unsigned low limb and signed high limb
__device__ __forceinline__ void split_limbs(int64_t d, uint32_t &lo, uint32_t &hi) {
    lo = (uint32_t)d & 0xFFFFFu;
    hi = (uint32_t)(d >> 20);
}

template <int DT, int K, bool UNIFORM>
__device__ __forceinline__ void deposit_row(uint32_t *cnt, int key, const typename Fmt<DT>::V v, int kt,
                                            int lane) {
    using Cfg = OnchipCfg<DT, K>;
    typename Fmt<DT>::Digit d[K];
    digits_of<DT, K>(v, kt, d);
    if (UNIFORM) {
        // small G: when the whole warp holds one group, reduce with a uniform REDUX first
        const int k0 = __shfl_sync(0xffffffffu, key, 0);
        if (__all_sync(0xffffffffu, key == k0 && key >= 0)) {
            uint32_t *p = cnt + (size_t)k0 * Cfg::CW;
#pragma unroll
            for (int l = 0; l < K; ++l) {
                if (Cfg::LIMBS == 2) {
                    uint32_t lo, hi;
                    split_limbs((int64_t)d[l], lo, hi);
                    lo = __reduce_add_sync(0xffffffffu, lo);
                    hi = __reduce_add_sync(0xffffffffu, hi);
                    if (lane == 0) { atomicAdd(p + 2 * l, lo); atomicAdd(p + 2 * l + 1, hi); }
                } else {
                    const uint32_t x = __reduce_add_sync(0xffffffffu, (uint32_t)(int32_t)d[l]);
                    if (lane == 0) atomicAdd(p + l, x);
                }
            }
            return;
        }
    }
    if (key < 0) return;
    uint32_t *p = cnt + (size_t)key * Cfg::CW;
#pragma unroll
    for (int l = 0; l < K; ++l) {
        if (Cfg::LIMBS == 2) {
            uint32_t lo, hi;
            split_limbs((int64_t)d[l], lo, hi);
            atomicAdd(p + 2 * l, lo);
            atomicAdd(p + 2 * l + 1, hi);
        } else {
            atomicAdd(p + l, (uint32_t)(int32_t)d[l]);
        }
    }
}

template <int DT, int K>
__device__ __forceinline__ int64_t counters_value(const uint32_t *c, int l) {
    if (Fmt<DT>::LIMBS == 2) return (int64_t)c[2 * l] + (int64_t)(int32_t)c[2 * l + 1] * (int64_t)(1 << 20);
    return (int64_t)(int32_t)c[l];
}

template <int DT, int K>
__global__ void __launch_bounds__(256)
k_onchip_accumulate(const int32_t *__restrict__ keys, const typename Fmt<DT>::V *__restrict__ vals,
                    int64_t n, int32_t G, int64_t chunk, int32_t *__restrict__ kglob,
                    unsigned long long *__restrict__ slots, uint32_t *__restrict__ status) {
    using F = Fmt<DT>;
    using V = typename F::V;
    using Cfg = OnchipCfg<DT, K>;
    constexpr int TPB = Cfg::TPB, R = Cfg::R, TILE = Cfg::TILE, CW = Cfg::CW;
    constexpr int NS = F::KMAX + K;  // absolute slots per group

    extern __shared__ __align__(16) unsigned char smem[];
    int64_t *tot = reinterpret_cast<int64_t *>(smem);                    // [G][K]
    uint32_t *cnt = reinterpret_cast<uint32_t *>(tot + (size_t)K * G);   // [G][CW]
    int32_t *ktop_cur = reinterpret_cast<int32_t *>(cnt + (size_t)CW * G);
    int32_t *ktop_next = ktop_cur + G;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    for (int i = tid; i < K * G; i += TPB) tot[i] = 0;
    for (int i = tid; i < CW * G; i += TPB) cnt[i] = 0;
    for (int i = tid; i < G; i += TPB) { ktop_cur[i] = 0; ktop_next[i] = 0; }
    __syncthreads();

    const bool small_g = G <= 32;
    const int64_t row0 = (int64_t)blockIdx.x * chunk;
    const int64_t row1 = min(n, row0 + chunk);
    uint32_t flags = 0;
    int since = 0;  // rows' worth of digits in the counters since the last fold

    for (int64_t base = row0; base < row1; base += TILE) {
        const int32_t *kp = keys + base + tid;
        const V *vp = vals + base + tid;
        const int rem = (int)min((int64_t)TILE, row1 - base) - tid;  // rows i*TPB < rem exist
        int32_t key[R];
        V val[R];
        int kc[R];
        // a1: coalesced loads (immediate offsets i*TPB from one base pointer)
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const bool in = i * TPB < rem;
            key[i] = in ? __ldg(kp + i * TPB) : -1;
            val[i] = in ? __ldg(vp + i * TPB) : V(0);
        }
        // a2: window tops; raise ktop_next of the row's group where needed
        int changed = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const bool in = i * TPB < rem;
            int k = key[i];
            const bool keyok = (uint32_t)k < (uint32_t)G;
            if (in && !keyok) flags |= FLAG_EKEY;
            const int ks = kstar_of<DT>(val[i], flags);
            const bool ok = in && keyok && ks >= 0;
            if (in && keyok && ks < 0) { /* EDOM / ERANGE already flagged */ }
            k = ok ? k : -1;
            const int cur = ok ? ktop_cur[k] : 0;
            if (ok && ks > cur) { atomicMax(&ktop_next[k], ks); changed = 1; }
            key[i] = k;
            kc[i] = cur;
        }
        const bool fold = since + TILE > Cfg::LIMIT;
        const int any = __syncthreads_or(changed);  // also: previous tile's deposits are done
        if (any || fold) {
            for (int g = tid; g < G; g += TPB) {
                uint32_t *c = cnt + (size_t)g * CW;
                int64_t *t = tot + (size_t)g * K;
                if (fold) {
#pragma unroll
                    for (int l = 0; l < K; ++l) t[l] += counters_value<DT, K>(c, l);
#pragma unroll
                    for (int j = 0; j < CW; ++j) c[j] = 0;
                }
                const int kn = ktop_next[g], ko = ktop_cur[g];
                if (kn != ko) {  // demotion by kn - ko levels
                    const int sh = kn - ko;
#pragma unroll
                    for (int l = K - 1; l >= 0; --l) {
                        const bool keep = l - sh >= 0;
                        t[l] = keep ? t[l - sh] : 0;
#pragma unroll
                        for (int b = 0; b < Cfg::LIMBS; ++b)
                            c[l * Cfg::LIMBS + b] = keep ? c[(l - sh) * Cfg::LIMBS + b] : 0u;
                    }
                    ktop_cur[g] = kn;
                }
            }
            __syncthreads();
            if (fold) since = 0;
            if (any) {
#pragma unroll
                for (int i = 0; i < R; ++i)
                    if (key[i] >= 0) kc[i] = ktop_cur[key[i]];
            }
        }
        since += TILE;

        // a3 + a4: digits under the group's current top, 32-bit shared atomics
        if (small_g) {
#pragma unroll
            for (int i = 0; i < R; ++i) deposit_row<DT, K, true>(cnt, key[i], val[i], kc[i], lane);
        } else {
#pragma unroll
            for (int i = 0; i < R; ++i) deposit_row<DT, K, false>(cnt, key[i], val[i], kc[i], lane);
        }
    }

    // flush: fold the counters, then publish the block's partial state into
    // the absolute-level slot table
    __syncthreads();
    for (int g = tid; g < G; g += TPB) {
        const int k = ktop_cur[g];
        if (k > 0) atomicMax(&kglob[g], k);
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const int64_t T = tot[(size_t)g * K + l] + counters_value<DT, K>(cnt + (size_t)g * CW, l);
            if (T != 0) {
                unsigned long long *p = slots + ((size_t)g * NS + (k - l + K - 1)) * 2;
                atomicAdd(p, (unsigned long long)(T & 0xFFFFFFFFll));
                atomicAdd(p + 1, (unsigned long long)(T >> 32));
            }
        }
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0 && flags) atomicOr(status, flags);
}

template <int DT, int K>
int launch_onchip(const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t *kglob,
                  unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
    using Cfg = OnchipCfg<DT, K>;
    auto kern = k_onchip_accumulate<DT, K>;
    const size_t smem = onchip_smem_bytes<DT, K>(G);
    if (smem > (size_t)device_props().smem_optin) return -1;
    static thread_local int configured_smem[2][5] = {};
    if (configured_smem[DT][K] < (int)smem) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return -2;
        configured_smem[DT][K] = (int)smem;
    }
    if (n == 0) return 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::TPB, smem);
    if (per_sm < 1) return -1;
    int64_t grid = (int64_t)per_sm * device_props().sms;
    // a block's int64 level sums must not overflow: <= 2^23 rows per block
    const int64_t min_grid = (n + (1ll << 23) - 1) >> 23;
    if (grid < min_grid) grid = min_grid;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = ((chunk + Cfg::TILE - 1) / Cfg::TILE) * Cfg::TILE;
    if (chunk > (1ll << 23)) chunk = 1ll << 23;
    grid = (n + chunk - 1) / chunk;
    kern<<<(unsigned)grid, Cfg::TPB, smem, st>>>(keys, (const typename Fmt<DT>::V *)vals, n, G, chunk,
                                                 kglob, slots, status);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int atomic_max_groups(int K, int DT) {
    const size_t cap = (size_t)device_props().smem_optin;
    size_t per = (size_t)(8 * K + 4 * K * (DT == 1 ? 2 : 1) + 8);  // == onchip_smem_bytes / G
    return (int)(cap / per);
}

// variant: 0 = auto (sorted where it fits), 1 = atomic, 2 = sorted.
// Initialised from REPRO_ONCHIP_VARIANT, settable through the C-ABI.
static int g_variant = -1;
static int onchip_variant() {
    if (g_variant < 0) {
        const char *e = getenv("REPRO_ONCHIP_VARIANT");
        g_variant = (e && e[0] == 'a') ? 1 : (e && e[0] == 's') ? 2 : 0;
    }
    return g_variant;
}
void set_onchip_variant(int v) { g_variant = (v >= 0 && v <= 2) ? v : 0; }

int onchip_max_groups(int K, int DT) {
    const int v = onchip_variant();
    if (v == 1) return atomic_max_groups(K, DT);
    if (v == 2) return sorted_max_groups(K, DT);
    return std::max(atomic_max_groups(K, DT), sorted_max_groups(K, DT));
}

int launch_onchip_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G,
                      int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                      int *launches) {
    const int v = onchip_variant();
    if (v != 1 && G <= sorted_max_groups(K, DT))
        return launch_sorted_any(DT, K, keys, vals, n, G, kglob, slots, status, st, launches);
    return launch_atomic_any(DT, K, keys, vals, n, G, kglob, slots, status, st, launches);
}

int launch_atomic_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G,
                      int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                      int *launches) {
#define ONCHIP_CASE(dt, k) \
    if (DT == dt && K == k) return launch_onchip<dt, k>(keys, vals, n, G, kglob, slots, status, st, launches);
    ONCHIP_CASE(1, 1) ONCHIP_CASE(1, 2) ONCHIP_CASE(1, 3) ONCHIP_CASE(1, 4)
    ONCHIP_CASE(0, 1) ONCHIP_CASE(0, 2) ONCHIP_CASE(0, 3) ONCHIP_CASE(0, 4)
#undef ONCHIP_CASE
    return -1;
}

}  // namespace repro
