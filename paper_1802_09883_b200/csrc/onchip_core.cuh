// onchip_core.cuh -- the per-row / per-table device code shared by the
// on-chip GroupBy kernel (k_onchip.cu) and the partitioned path's
// per-partition kernel (k_partition.cu).  See k_onchip.cu for the design.
#pragma once

#include "common.cuh"

namespace repro {

#ifndef ONCHIP_R64
#define ONCHIP_R64 15
#endif
#ifndef ONCHIP_MINBLOCKS
#define ONCHIP_MINBLOCKS 2
#endif
#ifndef ONCHIP_REGTOT_MAXG
#define ONCHIP_REGTOT_MAXG 1024
#endif

template <int DT, int K>
struct OnchipCfg {
    static constexpr int TPB = 256;
    static constexpr int R = (DT == 1) ? ONCHIP_R64 : 16;  // rows per thread per tile
    static constexpr int TILE = TPB * R;           // 3840 / 4096
    // limb counters accept at most LIMIT rows' worth of digits between folds
    static constexpr int LIMIT = (DT == 1) ? 4095 : 16383;
    static constexpr int LIMBS = Fmt<DT>::LIMBS;
    static constexpr int CW = K * LIMBS;  // 32-bit counters per group
    // group-major rows of CWP words; an odd stride spreads random groups over
    // all 32 banks (stride 6 would use only 16 and double the conflicts)
    static constexpr int CWP = CW | 1;
    static_assert(TILE <= LIMIT, "tile larger than limb headroom");
};

template <int DT, int K>
size_t onchip_smem_bytes(int G) {
    using C = OnchipCfg<DT, K>;
    return (size_t)G * (8 * K + 4 * C::CWP + 8) + 16;
}

// Limbs of one row's K digits, computed from the bits (common.cuh digits_of
// written out so that no 64-bit integer arithmetic is needed):
//   binary64: t = x (+) 1.5*2^52 has low word = low word of the digit d and
//   high word = high word of d + 0x43380000; limbs are d mod 2^20 and d >> 20
//   (a funnel shift of the two words).  binary32: one int32 limb per level.
// `s` is the row's value already scaled to units of the top level's ulp.
template <int DT, int K>
__device__ __forceinline__ void row_limbs(typename Fmt<DT>::V s, uint32_t (&lo)[K], uint32_t (&hi)[K]) {
    if (DT == 1) {
        const double M = 6755399441055744.0;       // 1.5 * 2^52
        const double T40 = 1099511627776.0;        // 2^40
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const double x = __hiloint2double(__double2hiint(s), __double2loint(s) | 1);
            const double t = __dadd_rn(x, M);
            const uint32_t tlo = (uint32_t)__double2loint(t);
            const uint32_t dhi = (uint32_t)__double2hiint(t) - 0x43380000u;
            lo[l] = tlo & 0xFFFFFu;
            hi[l] = __funnelshift_r(tlo, dhi, 20);
            if (l + 1 < K) s = __dmul_rn(__dsub_rn(s, __dsub_rn(t, M)), T40);
        }
    } else {
        const float M = 12582912.0f;               // 1.5 * 2^23
        const float T18 = 262144.0f;               // 2^18
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const float x = __uint_as_float(__float_as_uint((float)s) | 1u);
            const float t = __fadd_rn(x, M);
            lo[l] = __float_as_uint(t) - 0x4B400000u;
            hi[l] = 0;
            if (l + 1 < K) s = __fmul_rn(__fsub_rn((float)s, __fsub_rn(t, M)), T18);
        }
    }
}

template <int DT, int K, bool UNIFORM>
__device__ __forceinline__ void deposit_row(uint32_t *cnt, int key, typename Fmt<DT>::V s, int lane) {
    using Cfg = OnchipCfg<DT, K>;
    uint32_t lo[K], hi[K];
    row_limbs<DT, K>(s, lo, hi);
    if (UNIFORM) {
        // small G: when the whole warp holds one group, reduce with a uniform REDUX first
        const int k0 = __shfl_sync(0xffffffffu, key, 0);
        if (__all_sync(0xffffffffu, key == k0 && key >= 0)) {
            uint32_t *p = cnt + (size_t)k0 * Cfg::CWP;
#pragma unroll
            for (int l = 0; l < K; ++l) {
                const uint32_t a = __reduce_add_sync(0xffffffffu, lo[l]);
                if (Cfg::LIMBS == 2) {
                    const uint32_t b = __reduce_add_sync(0xffffffffu, hi[l]);
                    if (lane == 0) { atomicAdd(p + 2 * l, a); atomicAdd(p + 2 * l + 1, b); }
                } else if (lane == 0) {
                    atomicAdd(p + l, a);
                }
            }
            return;
        }
    }
    if (key >= 0) {
        uint32_t *p = cnt + (size_t)key * Cfg::CWP;
#pragma unroll
        for (int l = 0; l < K; ++l) {
            if (Cfg::LIMBS == 2) {
                atomicAdd(p + 2 * l, lo[l]);
                atomicAdd(p + 2 * l + 1, hi[l]);
            } else {
                atomicAdd(p + l, lo[l]);
            }
        }
    }
}

template <int DT, int K>
__device__ __forceinline__ int64_t counters_value(const uint32_t *c, int l) {
    if (Fmt<DT>::LIMBS == 2) return (int64_t)c[2 * l] + (int64_t)(int32_t)c[2 * l + 1] * (int64_t)(1 << 20);
    return (int64_t)(int32_t)c[l];
}

// Fold the limb counters of group g into its level sums t[] (if `fold`) and
// demote its levels when its window top moved.
template <int DT, int K>
__device__ __forceinline__ void fold_group(uint32_t *__restrict__ c, int64_t (&t)[K], bool fold, int32_t *ktop_cur,
                                           const int32_t *ktop_next, int g) {
    using Cfg = OnchipCfg<DT, K>;
    if (fold) {
#pragma unroll
        for (int l = 0; l < K; ++l) t[l] += counters_value<DT, K>(c, l);
#pragma unroll
        for (int w = 0; w < Cfg::CW; ++w) c[w] = 0;
    }
    const int kn = ktop_next[g], ko = ktop_cur[g];
    if (kn != ko) {
        const int sh = kn - ko;
#pragma unroll
        for (int r = 0; r < K; ++r) {  // sh single-level shifts (static register indices)
            if (r < sh) {
#pragma unroll
                for (int l = K - 1; l >= 1; --l) t[l] = t[l - 1];
                t[0] = 0;
            }
        }
#pragma unroll
        for (int l = K - 1; l >= 0; --l) {
#pragma unroll
            for (int b = 0; b < Cfg::LIMBS; ++b)
                c[l * Cfg::LIMBS + b] = l - sh >= 0 ? c[(l - sh) * Cfg::LIMBS + b] : 0u;
        }
        ktop_cur[g] = kn;
    }
}

// Publish a block's level sums of group g into the absolute-level slot table.
template <int DT, int K>
__device__ __forceinline__ void publish_group(const uint32_t *c, const int64_t (&t)[K], int k, int g,
                                              int32_t *kglob, unsigned long long *slots) {
    constexpr int NS = Fmt<DT>::KMAX + K;
    if (k > 0) atomicMax(&kglob[g], k);
#pragma unroll
    for (int l = 0; l < K; ++l) {
        const int64_t T = t[l] + counters_value<DT, K>(c, l);
        if (T != 0) {
            unsigned long long *p = slots + ((size_t)g * NS + (k - l + K - 1)) * 2;
            atomicAdd(p, (unsigned long long)(T & 0xFFFFFFFFll));
            atomicAdd(p + 1, (unsigned long long)(T >> 32));
        }
    }
}

// Level check of one row (Alg. 1 lines 3-9) without branches: error bits and
// the window top k*; returns the key, or -1 if the row does not deposit.
template <int DT>
__device__ __forceinline__ int check_row(int key, typename Fmt<DT>::V v, bool in, int G, uint32_t &flags,
                                         int &ks) {
    using F = Fmt<DT>;
    int be;
    if (DT == 1) be = ((uint32_t)__double2hiint((double)v) >> 20) & 0x7FF;
    else be = (__float_as_uint((float)v) >> 23) & 0xFF;
    const int t = max(be - F::BIAS + 2 + F::m - F::W, 0);
    ks = (t + F::W - 1) / F::W;
    const bool keyok = (uint32_t)key < (uint32_t)G;
    const uint32_t bad = !keyok ? FLAG_EKEY : (be == F::EXPMASK ? FLAG_EDOM : (ks > F::KMAX ? FLAG_ERANGE : 0u));
    flags |= in ? bad : 0u;
    return (in && bad == 0u) ? key : -1;
}

// Where a block's finished table goes: MODE 0 adds it into the absolute-level
// slot table (kglob, slots); MODE 1 writes it densely as one partial state per
// group (pk[g], pT[g*K + l]) for the partitioned path's merge.
struct PubArgs {
    int32_t *kglob;
    unsigned long long *slots;
    int32_t *pk;
    int64_t *pT;
};

// One block deposits rows [row0, row1) of (keys, vals) into a fresh table of G
// groups in shared memory (+ registers) and publishes it.  Must be entered by
// all threads of the block; `smem` is the dynamic shared memory.
template <int DT, int K, bool REGTOT, int MODE>
__device__ __forceinline__ void accumulate_range(const int32_t *__restrict__ keys,
                                                 const typename Fmt<DT>::V *__restrict__ vals, int64_t row0,
                                                 int64_t row1, int32_t G, unsigned char *smem, uint32_t &flags,
                                                 const PubArgs &out) {
    using F = Fmt<DT>;
    using V = typename F::V;
    using Cfg = OnchipCfg<DT, K>;
    constexpr int TPB = Cfg::TPB, R = Cfg::R, TILE = Cfg::TILE, CW = Cfg::CW, CWP = Cfg::CWP;
    constexpr int NS = F::KMAX + K;  // absolute slots per group
    constexpr int GPT = 4;           // groups per thread when the level sums live in registers

    int64_t *tot = reinterpret_cast<int64_t *>(smem);                    // [G][K] (unless REGTOT)
    uint32_t *cnt = reinterpret_cast<uint32_t *>(tot + (REGTOT ? 0 : (size_t)K * G));  // [G][CWP]
    int32_t *ktop_cur = reinterpret_cast<int32_t *>(cnt + (size_t)CWP * G);
    int32_t *ktop_next = ktop_cur + G;
    int32_t *kminmax = ktop_next + G;  // [0] min, [1] max of ktop_cur over the groups

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    int64_t treg[GPT][K];  // level sums of groups tid + j*TPB (REGTOT)
#pragma unroll
    for (int j = 0; j < GPT; ++j)
#pragma unroll
        for (int l = 0; l < K; ++l) treg[j][l] = 0;
    if (!REGTOT)
        for (int i = tid; i < K * G; i += TPB) tot[i] = 0;
    for (int i = tid; i < CWP * G; i += TPB) cnt[i] = 0;
    for (int i = tid; i < G; i += TPB) { ktop_cur[i] = 0; ktop_next[i] = 0; }
    __syncthreads();
    // block-uniform window top: when every group has the same top `kuni`,
    // rows need no per-group lookup (the common case after the first tiles)
    int kuni = 0;

    const bool small_g = G <= 32;
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
        if (kuni >= 0) {
#pragma unroll
            for (int i = 0; i < R; ++i) {
                int ks;
                const int k = check_row<DT>(key[i], val[i], i * TPB < rem, G, flags, ks);
                if (k >= 0 && ks > kuni) { atomicMax(&ktop_next[k], ks); changed = 1; }
                key[i] = k;
                kc[i] = kuni;
            }
        } else {
#pragma unroll
            for (int i = 0; i < R; ++i) {
                int ks;
                const int k = check_row<DT>(key[i], val[i], i * TPB < rem, G, flags, ks);
                const int cur = k >= 0 ? ktop_cur[k] : 0;
                if (k >= 0 && ks > cur) { atomicMax(&ktop_next[k], ks); changed = 1; }
                key[i] = k;
                kc[i] = cur;
            }
        }
        const bool fold = since + TILE > Cfg::LIMIT;
        const int any = __syncthreads_or(changed);  // also: previous tile's deposits are done
        if (any || fold) {
            // fold counters into the level sums and demote moved groups
            if (REGTOT) {
#pragma unroll
                for (int j = 0; j < GPT; ++j)
                    if (tid + j * TPB < G)
                        fold_group<DT, K>(cnt + (size_t)(tid + j * TPB) * CWP, treg[j], fold, ktop_cur, ktop_next,
                                          tid + j * TPB);
            } else {
                for (int g = tid; g < G; g += TPB) {
                    int64_t t[K];
#pragma unroll
                    for (int l = 0; l < K; ++l) t[l] = tot[(size_t)g * K + l];
                    fold_group<DT, K>(cnt + (size_t)g * CWP, t, fold, ktop_cur, ktop_next, g);
#pragma unroll
                    for (int l = 0; l < K; ++l) tot[(size_t)g * K + l] = t[l];
                }
            }
            if (any) {  // new block-uniform top?
                if (tid == 0) { kminmax[0] = 1 << 30; kminmax[1] = -1; }
                __syncthreads();
                int lo = 1 << 30, hi = -1;
                for (int g = tid; g < G; g += TPB) { lo = min(lo, ktop_cur[g]); hi = max(hi, ktop_cur[g]); }
                lo = __reduce_min_sync(0xffffffffu, lo);
                hi = __reduce_max_sync(0xffffffffu, hi);
                if (lane == 0) { atomicMin(&kminmax[0], lo); atomicMax(&kminmax[1], hi); }
            }
            __syncthreads();
            if (fold) since = 0;
            if (any) {
                kuni = kminmax[0] == kminmax[1] ? kminmax[1] : -1;
#pragma unroll
                for (int i = 0; i < R; ++i)
                    if (key[i] >= 0) kc[i] = ktop_cur[key[i]];
            }
        }
        since += TILE;

        // a3 + a4: digits under the group's current top, 32-bit shared atomics
        if (small_g) {
#pragma unroll
            for (int i = 0; i < R; ++i)
                deposit_row<DT, K, true>(cnt, key[i], F::mul(val[i], F::pow2(F::m - F::W * kc[i])), lane);
        } else if (kuni >= 0) {
            const V scale = F::pow2(F::m - F::W * kuni);
#pragma unroll
            for (int i = 0; i < R; ++i) deposit_row<DT, K, false>(cnt, key[i], F::mul(val[i], scale), lane);
        } else {
#pragma unroll
            for (int i = 0; i < R; ++i)
                deposit_row<DT, K, false>(cnt, key[i], F::mul(val[i], F::pow2(F::m - F::W * kc[i])), lane);
        }
    }

    // flush: fold the counters, then publish the block's table
    __syncthreads();
    auto pub = [&](int g, const int64_t(&t)[K]) {
        const uint32_t *c = cnt + (size_t)g * CWP;
        if (MODE == 0) {
            publish_group<DT, K>(c, t, ktop_cur[g], g, out.kglob, out.slots);
        } else {
            out.pk[g] = ktop_cur[g];
#pragma unroll
            for (int l = 0; l < K; ++l) out.pT[(size_t)g * K + l] = t[l] + counters_value<DT, K>(c, l);
        }
    };
    if (REGTOT) {
#pragma unroll
        for (int j = 0; j < GPT; ++j)
            if (tid + j * TPB < G) pub(tid + j * TPB, treg[j]);
    } else {
        for (int g = tid; g < G; g += TPB) {
            int64_t t[K];
#pragma unroll
            for (int l = 0; l < K; ++l) t[l] = tot[(size_t)g * K + l];
            pub(g, t);
        }
    }
    __syncthreads();  // the table may be re-initialised by the caller next
}


}  // namespace repro
