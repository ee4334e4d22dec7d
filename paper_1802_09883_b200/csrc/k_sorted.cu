// k_sorted.cu -- on-chip accumulate kernel with tile-level counting sort
// ("sorted" variant, the default on-chip path).
//
// Same job and same output as k_onchip_accumulate (k_onchip.cu): rows a1-a4/a6
// of SURVEY.md section 8 -- per row the window top k* (Alg. 1 lines 3-9,
// PAPER.md:658-665) and the K integer digits (lines 10-16), added into the
// block's shared-memory table of group states, whose int64 level sums are
// published into the absolute-level slot table at the end.
//
// Why a sort: shared-memory atomics cost ~4.3 cycles per warp instruction on
// sm_100a whatever the address pattern (measured, scripts/microbench.cu), and
// a binary64 row needs 2K of them (20-bit limbs).  So each tile of rows is
// first grouped by key with a counting sort in shared memory (one histogram
// atomic per row), then every thread walks R consecutive sorted rows and
// accumulates each run of equal keys in registers.  A run strictly inside a
// thread's segment belongs to that thread alone: it is added to the table
// with plain loads/stores.  Only the first and last run of a segment can be
// shared with a neighbour; those two are added with limb atomics after the
// loop, by all lanes together.  Integer addition is associative, so the order
// in which runs land does not matter (the reason the paper's type can be used
// under any physical order).
//
// Alg. 1's level check stays a tile-phase integer max (see k_onchip.cu), and
// limb counters are folded into the int64 sums before they can overflow.
#include "common.cuh"
#include "internal.h"

namespace repro {

template <int DT, int K>
struct SortCfg {
    static constexpr int TPB = 256;
    static constexpr int R = (DT == 1) ? 15 : 16;  // rows per thread per tile
    static constexpr int TILE = TPB * R;           // 3840 / 4096
    static constexpr int LIMIT = (DT == 1) ? 4095 : 16383;  // limb headroom (additions of mass)
    static constexpr int NL = Fmt<DT>::LIMBS;
    static constexpr int KP = (K == 3) ? 4 : K;   // padded int64 sums per group
    static constexpr int CW = K * NL;             // 32-bit counters per group
    static_assert(TILE <= LIMIT, "tile larger than limb headroom");
};

// shared-memory layout, identical on host (size) and device (carve)
template <int DT, int K>
struct SortLayout {
    size_t tot, cnt, kcur, knext, bins, wsum, sval, skey, bytes;
    int GB;  // bins per buffer (G + 1 rounded up to even)
    __host__ __device__ SortLayout(int G) {
        using C = SortCfg<DT, K>;
        GB = (G + 2) & ~1;
        size_t o = 0;
        tot = o;   o += (size_t)8 * C::KP * G;
        cnt = o;   o += (size_t)4 * C::CW * G;
        o = (o + 7) & ~(size_t)7;
        kcur = o;  o += (size_t)4 * G;
        knext = o; o += (size_t)4 * G;
        bins = o;  o += (size_t)4 * 2 * GB;
        wsum = o;  o += 4 * 32;
        o = (o + 15) & ~(size_t)15;
        sval = o;  o += sizeof(typename Fmt<DT>::V) * C::TILE;
        skey = o;  o += 2 * C::TILE;
        bytes = (o + 15) & ~(size_t)15;
    }
};

template <int DT, int K>
__device__ __forceinline__ void flush_atomic(uint32_t *cnt, int key, const int64_t (&acc)[K], bool valid, int lane) {
    using C = SortCfg<DT, K>;
    // warp-uniform group (small G / heavy skew): reduce first, one lane adds
    const int k0 = __shfl_sync(0xffffffffu, key, 0);
    const bool uni = __all_sync(0xffffffffu, valid && key == k0);
    uint32_t *p = cnt + (size_t)(uni ? k0 : key) * C::CW;
#pragma unroll
    for (int l = 0; l < K; ++l) {
        uint32_t a, b = 0;
        if (C::NL == 2) {
            a = (uint32_t)((uint64_t)acc[l] & 0xFFFFFull);
            b = (uint32_t)(int32_t)(acc[l] >> 20);
        } else {
            a = (uint32_t)(int32_t)acc[l];
        }
        if (uni) {
            a = __reduce_add_sync(0xffffffffu, a);
            if (C::NL == 2) b = __reduce_add_sync(0xffffffffu, b);
            if (lane == 0) {
                atomicAdd(p + l * C::NL, a);
                if (C::NL == 2) atomicAdd(p + l * C::NL + 1, b);
            }
        } else if (valid) {
            atomicAdd(p + l * C::NL, a);
            if (C::NL == 2) atomicAdd(p + l * C::NL + 1, b);
        }
    }
}

template <int DT, int K>
__device__ __forceinline__ int64_t limbs_value(const uint32_t *c) {
    using C = SortCfg<DT, K>;
    if (C::NL == 2) return (int64_t)c[0] + (int64_t)(int32_t)c[1] * (int64_t)(1 << 20);
    return (int64_t)(int32_t)c[0];
}

template <int DT, int K>
__global__ void __launch_bounds__(256, 2)
k_onchip_sorted(const int32_t *__restrict__ keys, const typename Fmt<DT>::V *__restrict__ vals, int64_t n,
                int32_t G, int64_t chunk, int32_t *__restrict__ kglob, unsigned long long *__restrict__ slots,
                uint32_t *__restrict__ status) {
    using F = Fmt<DT>;
    using V = typename F::V;
    using C = SortCfg<DT, K>;
    constexpr int TPB = C::TPB, R = C::R, TILE = C::TILE, KP = C::KP, CW = C::CW;
    constexpr int NS = F::KMAX + K;

    extern __shared__ __align__(16) unsigned char smem[];
    const SortLayout<DT, K> L(G);
    int64_t *tot = reinterpret_cast<int64_t *>(smem + L.tot);
    uint32_t *cnt = reinterpret_cast<uint32_t *>(smem + L.cnt);
    int32_t *ktop_cur = reinterpret_cast<int32_t *>(smem + L.kcur);
    int32_t *ktop_next = reinterpret_cast<int32_t *>(smem + L.knext);
    uint32_t *bins = reinterpret_cast<uint32_t *>(smem + L.bins);
    uint32_t *wsum = reinterpret_cast<uint32_t *>(smem + L.wsum);
    V *sval = reinterpret_cast<V *>(smem + L.sval);
    uint16_t *skey = reinterpret_cast<uint16_t *>(smem + L.skey);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < KP * G; i += TPB) tot[i] = 0;
    for (int i = tid; i < CW * G; i += TPB) cnt[i] = 0;
    for (int i = tid; i < G; i += TPB) { ktop_cur[i] = 0; ktop_next[i] = 0; }
    for (int i = tid; i < 2 * L.GB; i += TPB) bins[i] = 0;
    __syncthreads();

    // scan chunk of this thread over the G+1 bins
    const int cper = (G + 1 + TPB - 1) / TPB;
    const int s0 = min(tid * cper, G + 1), s1 = min(s0 + cper, G + 1);

    const int64_t row0 = (int64_t)blockIdx.x * chunk;
    const int64_t row1 = min(n, row0 + chunk);
    uint32_t flags = 0;
    int since = 0, buf = 0;

    for (int64_t base = row0; base < row1; base += TILE, buf ^= 1) {
        uint32_t *bin = bins + buf * L.GB;
        int32_t key[R];
        V val[R];
        uint32_t rank[R];
        int changed = 0;
        // ---- P0: load, validate, level check, histogram ------------------
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int64_t r = base + (int64_t)i * TPB + tid;
            int k = G;
            V v = V(0);
            if (r < row1) {
                k = __ldg(keys + r);
                v = __ldg(vals + r);
                if ((uint32_t)k >= (uint32_t)G) {
                    flags |= FLAG_EKEY;
                    k = G;
                } else {
                    const int ks = kstar_of<DT>(v, flags);
                    if (ks < 0) {
                        k = G;
                    } else if (ks > ktop_cur[k]) {
                        atomicMax(&ktop_next[k], ks);
                        changed = 1;
                    }
                }
            }
            key[i] = k;
            val[i] = v;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int k0 = __shfl_sync(0xffffffffu, key[i], 0);
            if (__all_sync(0xffffffffu, key[i] == k0)) {
                uint32_t b0 = 0;
                if (lane == 0) b0 = atomicAdd(&bin[k0], 32u);
                rank[i] = __shfl_sync(0xffffffffu, b0, 0) + lane;
            } else {
                rank[i] = atomicAdd(&bin[key[i]], 1u);
            }
        }
        const bool fold = since + TILE > C::LIMIT;
        const int any = __syncthreads_or(changed);  // B1: histogram complete, previous tile done
        // ---- P1: fold limb counters / demote levels / scan bins ----------
        if (fold || any) {
            for (int g = tid; g < G; g += TPB) {
                if (fold) {
#pragma unroll
                    for (int l = 0; l < K; ++l) {
                        uint32_t *c = cnt + (size_t)g * CW + l * C::NL;
                        tot[(size_t)g * KP + l] += limbs_value<DT, K>(c);
                        c[0] = 0;
                        if (C::NL == 2) c[1] = 0;
                    }
                }
                const int kn = ktop_next[g], ko = ktop_cur[g];
                if (kn != ko) {  // demotion by kn - ko levels
                    const int sh = kn - ko;
#pragma unroll
                    for (int l = K - 1; l >= 0; --l) {
                        const bool keep = l - sh >= 0;
                        tot[(size_t)g * KP + l] = keep ? tot[(size_t)g * KP + l - sh] : 0;
#pragma unroll
                        for (int b = 0; b < C::NL; ++b)
                            cnt[(size_t)g * CW + l * C::NL + b] = keep ? cnt[(size_t)g * CW + (l - sh) * C::NL + b] : 0u;
                    }
                    ktop_cur[g] = kn;
                }
            }
        }
        if (fold) since = 0;
        since += TILE;
        uint32_t local = 0;
        for (int j = s0; j < s1; ++j) {
            const uint32_t t = bin[j];
            bin[j] = local;
            local += t;
        }
        uint32_t incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();  // B2
        uint32_t prefix = incl - local;
        for (int w = 0; w < warp; ++w) prefix += wsum[w];
        for (int j = s0; j < s1; ++j) bin[j] += prefix;
        __syncthreads();  // B3
        // ---- P2: scatter rows into key order ------------------------------
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const uint32_t pos = bin[key[i]] + rank[i];
            skey[pos] = (uint16_t)key[i];
            sval[pos] = val[i];
        }
        __syncthreads();  // B4
        for (int j = s0; j < s1; ++j) bin[j] = 0;  // ready for tile t+2
        // ---- P3: runs of equal keys, digits, accumulate ------------------
        const int p0 = tid * R;
        int64_t acc[K], facc[K];
        int cur = -1, fkey = -1;
        bool infirst = true;
#pragma unroll
        for (int l = 0; l < K; ++l) { acc[l] = 0; facc[l] = 0; }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int k = skey[p0 + i];
            const V v = sval[p0 + i];
            const bool valid = k < G;
            typename F::Digit d[K];
            digits_of<DT, K>(v, valid ? ktop_cur[k] : 0, d);
            if (k != cur) {
                if (cur >= 0) {
                    if (infirst) {
#pragma unroll
                        for (int l = 0; l < K; ++l) facc[l] = acc[l];
                        fkey = cur;
                    } else {  // interior run: this thread owns the group in this tile
                        int64_t *t = tot + (size_t)cur * KP;
#pragma unroll
                        for (int l = 0; l < K; ++l) t[l] += acc[l];
                    }
                    infirst = false;
                }
#pragma unroll
                for (int l = 0; l < K; ++l) acc[l] = 0;
                cur = valid ? k : -1;
            }
            if (valid) {
#pragma unroll
                for (int l = 0; l < K; ++l) acc[l] += (int64_t)d[l];
            }
        }
        // first and last run of the segment may be shared: atomics, all lanes together
        flush_atomic<DT, K>(cnt, cur, acc, cur >= 0, lane);
        flush_atomic<DT, K>(cnt, fkey, facc, fkey >= 0, lane);
    }

    // publish the block's partial state into the absolute-level slot table
    __syncthreads();
    for (int g = tid; g < G; g += TPB) {
        const int k = ktop_cur[g];
        if (k > 0) atomicMax(&kglob[g], k);
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const int64_t T = tot[(size_t)g * KP + l] + limbs_value<DT, K>(cnt + (size_t)g * CW + l * C::NL);
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
size_t sorted_smem_bytes(int G) {
    return SortLayout<DT, K>(G).bytes;
}

template <int DT, int K>
int launch_sorted(const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t *kglob,
                  unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
    using C = SortCfg<DT, K>;
    auto kern = k_onchip_sorted<DT, K>;
    const size_t smem = sorted_smem_bytes<DT, K>(G);
    if (G > 65535 || smem > (size_t)device_props().smem_optin) return -1;
    static thread_local int configured[2][5] = {};
    if (configured[DT][K] < (int)smem) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return -2;
        configured[DT][K] = (int)smem;
    }
    if (n == 0) return 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::TPB, smem);
    if (per_sm < 1) return -1;
    int64_t grid = (int64_t)per_sm * device_props().sms;
    const int64_t min_grid = (n + (1ll << 23) - 1) >> 23;  // <= 2^23 rows per block (int64 sums)
    if (grid < min_grid) grid = min_grid;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = ((chunk + C::TILE - 1) / C::TILE) * C::TILE;
    if (chunk > (1ll << 23)) chunk = (1ll << 23) / C::TILE * C::TILE;
    grid = (n + chunk - 1) / chunk;
    kern<<<(unsigned)grid, C::TPB, smem, st>>>(keys, (const typename Fmt<DT>::V *)vals, n, G, chunk, kglob, slots,
                                               status);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int sorted_max_groups(int K, int DT) {
    const size_t cap = (size_t)device_props().smem_optin;
    int lo = 1, hi = 65535;
    auto fits = [&](int G) -> bool {
        size_t b = 0;
#define SZ(dt, k) \
    if (DT == dt && K == k) b = sorted_smem_bytes<dt, k>(G);
        SZ(1, 1) SZ(1, 2) SZ(1, 3) SZ(1, 4) SZ(0, 1) SZ(0, 2) SZ(0, 3) SZ(0, 4)
#undef SZ
        return b != 0 && b <= cap;
    };
    if (!fits(1)) return 0;
    while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (fits(mid)) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

int launch_sorted_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t *kglob,
                      unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
#define SORTED_CASE(dt, k) \
    if (DT == dt && K == k) return launch_sorted<dt, k>(keys, vals, n, G, kglob, slots, status, st, launches);
    SORTED_CASE(1, 1) SORTED_CASE(1, 2) SORTED_CASE(1, 3) SORTED_CASE(1, 4)
    SORTED_CASE(0, 1) SORTED_CASE(0, 2) SORTED_CASE(0, 3) SORTED_CASE(0, 4)
#undef SORTED_CASE
    return -1;
}

}  // namespace repro
