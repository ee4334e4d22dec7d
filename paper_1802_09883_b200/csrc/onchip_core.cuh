// onchip_core.cuh -- the per-row / per-table device code shared by the
// on-chip GroupBy kernel (k_onchip.cu) and the partitioned path's
// per-partition kernel (k_partition.cu).  See k_onchip.cu for the design.
#pragma once

#include "common.cuh"

namespace repro {

#ifndef ONCHIP_R64
#define ONCHIP_R64 7
#endif
#ifndef ONCHIP_R32
#define ONCHIP_R32 15
#endif
#ifndef ONCHIP_MINBLOCKS
#define ONCHIP_MINBLOCKS 2
#endif
#ifndef ONCHIP_STAGES
#define ONCHIP_STAGES 3
#endif
#ifndef ONCHIP_FAST
#define ONCHIP_FAST 1
#endif
#ifndef ONCHIP_SKIPZ
#define ONCHIP_SKIPZ 1
#endif
#ifndef ONCHIP_SMALLG
#define ONCHIP_SMALLG 0  // groups up to which the generic path's warp-uniform REDUX is used
#endif
#ifndef ONCHIP_LANEREP
#define ONCHIP_LANEREP 32  // groups up to which the counters have one copy per lane (<= LANE_G)
#endif
#ifndef ONCHIP_RMULTI
#define ONCHIP_RMULTI 2  // input rows per thread per tile of the multi-column sources
#endif
#ifndef ONCHIP_NB
#define ONCHIP_NB 4
#endif
#ifndef ONCHIP_PRED
#define ONCHIP_PRED 0  // 1: lanes whose limb is zero skip the atomic (predicated, no branch)
#endif
#ifndef ONCHIP_DYNFOLD
#define ONCHIP_DYNFOLD 1  // 1: fast-path atomics return the old counter; fold only when one nears 2^30
#endif

// Table geometry.  The limb counters are WORD-MAJOR: counter w of group g is
// cnt[w * GQ + g], with GQ the group count rounded up to a multiple of 4 (1024
// when the level sums live in registers, so every address offset is an
// immediate).  A warp's shared atomic on one counter position w then hits
// bank (g + const) mod 32 -- random groups spread over all banks -- while the
// fold reads and clears four groups' counters with one 128-bit access.
template <int DT, int K>
struct OnchipCfg {
    static constexpr int TPB = 256;
    static constexpr int R = (DT == 1) ? ONCHIP_R64 : ONCHIP_R32;  // rows per thread per tile
    static constexpr int TILE = TPB * R;
    // limb counters accept at most LIMIT rows' worth of digits between folds:
    // balanced binary64 limbs have |limb| <= 2^19 (4095 * 2^19 < 2^31), binary32
    // digits |d| <= 2^17 (16383 * 2^17 < 2^31)
    static constexpr int LIMIT = (DT == 1) ? 4095 : 16383;
    static constexpr int LIMBS = Fmt<DT>::LIMBS;
    static constexpr int CW = K * LIMBS;  // 32-bit counters per group
    static constexpr int REG_GQ = 4 * TPB;  // groups covered when level sums are in registers (4 per thread)
    // small G (<= LANE_G): one counter copy per lane -- counter w of group g
    // for lane l at cnt[w * REG_GQ + 32 g + l], always bank l -- because 32
    // lanes adding to a few shared words serialise; level sums in shared
    // memory per counter word (int64 [LANE_G][CW])
    static constexpr int LANE_G = REG_GQ / 32;
    static_assert(TILE <= LIMIT, "tile larger than limb headroom");
};

// groups per counter row: REG_GQ with register level sums, else G rounded to 4
template <int DT, int K>
__host__ __device__ inline int onchip_gq(int G, bool regtot) {
    return regtot ? OnchipCfg<DT, K>::REG_GQ : (G + 3) & ~3;
}

// Shared memory of one block: [level sums int64 [GQ][K] (unless REGTOT)]
// [counters u32 [CW][GQ]] [ktop_cur [GQ]] [ktop_next [GQ]] [16 words misc]
// [REGTOT: lane-copy level sums int64 [LANE_G][CW]],
// then, for the TMA-fed kernel, 128 bytes of mbarriers and a ring of STAGES
// tiles of keys + values.
template <int DT, int K>
__host__ __device__ inline size_t onchip_table_bytes(int G, bool regtot = false) {
    using C = OnchipCfg<DT, K>;
    const size_t gq = (size_t)onchip_gq<DT, K>(G, regtot);
    return gq * ((regtot ? 0 : 8 * K) + 4 * C::CW + 8) + 64 + (regtot ? (size_t)8 * C::LANE_G * C::CW : 0);
}
template <int DT, int K, int NCOL = 1, int RIN = OnchipCfg<DT, K>::R>
constexpr size_t onchip_ring_bytes() {
    using C = OnchipCfg<DT, K>;
    return 128 + (size_t)ONCHIP_STAGES * C::TPB * RIN * (4 + NCOL * sizeof(typename Fmt<DT>::V));
}
template <int DT, int K>
size_t onchip_smem_bytes(int G, bool regtot = false, bool tma = false) {
    return ((onchip_table_bytes<DT, K>(G, regtot) + 127) & ~(size_t)127) + (tma ? onchip_ring_bytes<DT, K>() : 0);
}

// ---- TMA bulk copies (cp.async.bulk) and mbarriers -------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        :: "r"(bar), "r"(parity) : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both 16-B aligned),
// completing on mbarrier `bar`
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Bitwise OR of v over the block; also a full barrier.  __syncthreads_or only
// says whether ANY thread's predicate was non-zero (it returns 1, not the OR
// of the values), so multi-bit flags go through a shared word.  Three words
// rotate: the word of call c + 1 is cleared in call c, after every thread
// has read it in call c - 2 (before the barrier of call c - 1).
struct BlockOr {
    int *w;    // 3 shared words, zeroed before the first call (and a barrier)
    int call;  // calls so far (block-uniform)
    __device__ __forceinline__ int operator()(int v) {
        const int p = call % 3;
        if (threadIdx.x == 0) w[(p + 1) % 3] = 0;
        v = __reduce_or_sync(0xffffffffu, v);
        if ((threadIdx.x & 31) == 0 && v) atomicOr(&w[p], v);
        __syncthreads();
        ++call;
        return *(volatile int *)&w[p];
    }
};

// Limbs of one row's K digits, computed from the bits (common.cuh digits_of
// written out so that no 64-bit integer arithmetic is needed).
//   binary64: the extractor is M' = 1.5*2^52 + 2^19, so t = x (+) M' has the
//   bits of 1.5*2^52 plus (d + 2^19) (an integer shift of the extractor does
//   not change the rounding of x, and t (-) M' = d exactly).  The digit is split
//   into BALANCED limbs d = lo + hi*2^20 with lo = ((d + 2^19) mod 2^20) - 2^19
//   in [-2^19, 2^19) and hi = floor((d + 2^19) / 2^20) in [-2^19, 2^19]: a
//   digit with |d| < 2^19 has hi == 0 whatever its sign, a multiple of 2^20 has
//   lo == 0 (deposit_batch skips counters that a whole warp leaves at zero).
//   hi is a funnel shift of the two words of t (the exponent field of t
//   contributes exactly 0x80000000 to it).
//   binary32: one int32 limb per level (|d| <= 2^17).
// `s` is the row's value already scaled to units of the top level's ulp.
template <int DT, int K>
__device__ __forceinline__ void row_limbs(typename Fmt<DT>::V s, uint32_t (&lo)[K], uint32_t (&hi)[K]) {
    if (DT == 1) {
        const double M = 6755399441055744.0 + 524288.0;  // 1.5 * 2^52 + 2^19
        const double T40 = 1099511627776.0;              // 2^40
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const double x = __hiloint2double(__double2hiint(s), __double2loint(s) | 1);
            const double t = __dadd_rn(x, M);
            const uint32_t tlo = (uint32_t)__double2loint(t);
            const uint32_t thi = (uint32_t)__double2hiint(t);
            lo[l] = (tlo & 0xFFFFFu) - 0x80000u;
            hi[l] = __funnelshift_r(tlo, thi, 20) ^ 0x80000000u;
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

// 32-bit shared-memory reduction (ATOMS.ADD without return) at a shared-window
// address.
__device__ __forceinline__ void red_shared(uint32_t a, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(a), "r"(v) : "memory");
}
// the same, returning the counter's old value folded into `big`: bit 31 of
// big is set once any observed counter has |old| >= 2^30 (bits 31 and 30
// differ), the trigger of the dynamic fold (ONCHIP_DYNFOLD)
__device__ __forceinline__ void red_shared_obs(uint32_t a, uint32_t v, uint32_t &big) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
    big |= old ^ (old << 1);
}
// the same, predicated off for a zero addend (a lane that adds nothing does
// not take part in the bank access)
__device__ __forceinline__ void red_shared_nz(uint32_t a, uint32_t v) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p red.shared.add.u32 [%0], %1;\n\t}"
                 :: "r"(a), "r"(v) : "memory");
}

// Generic deposit of one row: digits under the window whose scale is already
// applied to s; key < 0 deposits nothing.  UNIFORM (small G): a warp whose
// lanes all hold one group reduces with REDUX first.
template <int DT, int K, bool UNIFORM, bool OBS = false>
__device__ __forceinline__ void deposit_row(uint32_t *cnt, int gq, int key, typename Fmt<DT>::V s, int lane,
                                            uint32_t *big = nullptr) {
    using Cfg = OnchipCfg<DT, K>;
    uint32_t lo[K], hi[K];
    row_limbs<DT, K>(s, lo, hi);
    if (UNIFORM) {
        const int k0 = __shfl_sync(0xffffffffu, key, 0);
        if (__all_sync(0xffffffffu, key == k0 && key >= 0)) {
            uint32_t *p = cnt + k0;
#pragma unroll
            for (int l = 0; l < K; ++l) {
                const uint32_t a = __reduce_add_sync(0xffffffffu, lo[l]);
                if (Cfg::LIMBS == 2) {
                    const uint32_t b = __reduce_add_sync(0xffffffffu, hi[l]);
                    if (lane == 0) {
                        atomicAdd(p + (size_t)(2 * l) * gq, a);
                        atomicAdd(p + (size_t)(2 * l + 1) * gq, b);
                    }
                } else if (lane == 0) {
                    atomicAdd(p + (size_t)l * gq, a);
                }
            }
            return;
        }
    }
    if (key >= 0) {
        uint32_t *p = cnt + key;
#pragma unroll
        for (int l = 0; l < K; ++l) {
#pragma unroll
            for (int h = 0; h < Cfg::LIMBS; ++h) {
                uint32_t *c = p + (size_t)(Cfg::LIMBS * l + h) * gq;
                const uint32_t v = h ? hi[l] : lo[l];
                if (OBS) red_shared_obs((uint32_t)__cvta_generic_to_shared(c), v, *big);
                else atomicAdd(c, v);
            }
        }
    }
}

// Per-level extractors of the fast path for window top k: level l (ulp u,
// the top level is l = 0) uses E_l = 1.5 * 2^m * u (+ 2^19 u for binary64's
// balanced limbs).  x (+) E_l for an unscaled remainder x is the paper's own
// extraction step q = (r (+) S) (-) S (Alg. 1 line 11) with S = E_l,
// and the bits of the sum are those of 1.5 * 2^m * u plus the digit: no scaling
// multiplies are needed.  `eb` holds the high word of 1.5 * 2^m * u shifted
// left by 12 (binary64: removed from the funnel-shifted high limb) or the
// bits of 1.5 * 2^m * u (binary32).
template <int DT, int K>
struct Extractors {
    typename Fmt<DT>::V e[K];
    uint32_t eb[K];
    __device__ __forceinline__ Extractors(int k) {
        using F = Fmt<DT>;
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const int ue = F::W * (k - l) - F::m;  // log2 of the level's ulp
            const typename F::V base = F::add(F::pow2(ue + F::m), F::pow2(ue + F::m - 1));  // 1.5 * 2^m * u
            if (DT == 1) {
                e[l] = F::add(base, F::pow2(ue + 19));
                eb[l] = (uint32_t)(F::bits(base) >> 32) << 12;
            } else {
                e[l] = base;
                eb[l] = (uint32_t)F::bits(base);
            }
        }
    }
};

// Fast-path deposit of NB rows known to be valid (keys in range, k* <= the
// block-uniform top): all limbs of the batch are computed first, then each
// counter position is updated for every row of the batch unless the whole warp
// holds zeros there (one vote per position and batch: small digits and values
// with few significant bits leave whole counters untouched).  Counter w of
// group g lives at shared address cbase + g * kstride + w * wstride.
template <int DT, int K, int NB, bool OBS>
__device__ __forceinline__ void deposit_batch(uint32_t cbase, uint32_t kstride, uint32_t wstride, const int32_t *key,
                                              const typename Fmt<DT>::V *val, const Extractors<DT, K> &ex,
                                              uint32_t &big) {
    using Cfg = OnchipCfg<DT, K>;
    uint32_t lo[NB][K], hi[NB][K], a[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        a[i] = cbase + kstride * (uint32_t)key[i];
        if (DT == 1) {
            double r = (double)val[i];
#pragma unroll
            for (int l = 0; l < K; ++l) {
                const double x = __hiloint2double(__double2hiint(r), __double2loint(r) | 1);  // reading A-1
                const double t = __dadd_rn(x, (double)ex.e[l]);
                const uint32_t tlo = (uint32_t)__double2loint(t);
                const uint32_t thi = (uint32_t)__double2hiint(t);
                lo[i][l] = (tlo & 0xFFFFFu) - 0x80000u;
                hi[i][l] = __funnelshift_r(tlo, thi, 20) - ex.eb[l];
                if (l + 1 < K) r = __dsub_rn(r, __dsub_rn(t, (double)ex.e[l]));
            }
        } else {
            float r = (float)val[i];
#pragma unroll
            for (int l = 0; l < K; ++l) {
                const float x = __uint_as_float(__float_as_uint(r) | 1u);
                const float t = __fadd_rn(x, (float)ex.e[l]);
                lo[i][l] = __float_as_uint(t) - ex.eb[l];
                hi[i][l] = 0;
                if (l + 1 < K) r = __fsub_rn(r, __fsub_rn(t, (float)ex.e[l]));
            }
        }
    }
#pragma unroll
    for (int l = 0; l < K; ++l) {
#pragma unroll
        for (int h = 0; h < Cfg::LIMBS; ++h) {
            uint32_t any = 0;
#pragma unroll
            for (int i = 0; i < NB; ++i) any |= h ? hi[i][l] : lo[i][l];
            if (ONCHIP_PRED == 1) {
                const uint32_t off = (uint32_t)(Cfg::LIMBS * l + h) * wstride;
#pragma unroll
                for (int i = 0; i < NB; ++i) red_shared_nz(a[i] + off, h ? hi[i][l] : lo[i][l]);
            } else if (ONCHIP_SKIPZ == 0 || __any_sync(0xffffffffu, any != 0u)) {
                const uint32_t off = (uint32_t)(Cfg::LIMBS * l + h) * wstride;
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    if (OBS) red_shared_obs(a[i] + off, h ? hi[i][l] : lo[i][l], big);
                    else if (ONCHIP_PRED == 2) red_shared_nz(a[i] + off, h ? hi[i][l] : lo[i][l]);
                    else red_shared(a[i] + off, h ? hi[i][l] : lo[i][l]);
                }
            }
        }
    }
}

// value of one level's counters (low and high limb counter words)
template <int DT, int K>
__device__ __forceinline__ int64_t limbs_value(uint32_t clo, uint32_t chi) {
    if (Fmt<DT>::LIMBS == 2) return (int64_t)(int32_t)clo + (int64_t)(int32_t)chi * (int64_t)(1 << 20);
    return (int64_t)(int32_t)clo;
}
template <int DT, int K>
__device__ __forceinline__ int64_t counters_value(const uint32_t *cnt, int gq, int g, int l) {
    if (Fmt<DT>::LIMBS == 2)
        return limbs_value<DT, K>(cnt[(size_t)(2 * l) * gq + g], cnt[(size_t)(2 * l + 1) * gq + g]);
    return limbs_value<DT, K>(cnt[(size_t)l * gq + g], 0u);
}

// Fold the limb counters of the four groups 4q..4q+3 into their level sums
// t[4][K] (if `fold`: one 128-bit load and store per counter position) and
// demote the groups whose window top moved (ktop_next > ktop_cur, PAPER.md:
// 661-664): level sums and counters shift down by the difference, the top
// level restarts at zero.
template <int DT, int K>
__device__ __forceinline__ void fold_quad(uint32_t *__restrict__ cnt, int gq, int q, int64_t (&t)[4][K], bool fold,
                                          int32_t *ktop_cur, const int32_t *ktop_next) {
    using Cfg = OnchipCfg<DT, K>;
    if (fold) {
        uint4 c[Cfg::CW];
#pragma unroll
        for (int w = 0; w < Cfg::CW; ++w) {
            uint4 *p = reinterpret_cast<uint4 *>(cnt + (size_t)w * gq) + q;
            c[w] = *p;
            *p = make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int l = 0; l < K; ++l) {
            const uint4 a = c[Cfg::LIMBS * l];
            const uint4 b = Cfg::LIMBS == 2 ? c[Cfg::LIMBS * l + 1] : make_uint4(0u, 0u, 0u, 0u);
            t[0][l] += limbs_value<DT, K>(a.x, b.x);
            t[1][l] += limbs_value<DT, K>(a.y, b.y);
            t[2][l] += limbs_value<DT, K>(a.z, b.z);
            t[3][l] += limbs_value<DT, K>(a.w, b.w);
        }
    }
    const int4 kn = reinterpret_cast<const int4 *>(ktop_next)[q];
    const int4 ko = reinterpret_cast<const int4 *>(ktop_cur)[q];
    if (kn.x != ko.x || kn.y != ko.y || kn.z != ko.z || kn.w != ko.w) {
        const int knv[4] = {kn.x, kn.y, kn.z, kn.w}, kov[4] = {ko.x, ko.y, ko.z, ko.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int sh = knv[j] - kov[j];
            if (sh == 0) continue;
            const int g = 4 * q + j;
#pragma unroll
            for (int r = 0; r < K; ++r) {  // sh single-level shifts (static register indices)
                if (r < sh) {
#pragma unroll
                    for (int l = K - 1; l >= 1; --l) t[j][l] = t[j][l - 1];
                    t[j][0] = 0;
                }
            }
#pragma unroll
            for (int l = K - 1; l >= 0; --l) {
#pragma unroll
                for (int b = 0; b < Cfg::LIMBS; ++b)
                    cnt[(size_t)(l * Cfg::LIMBS + b) * gq + g] =
                        l - sh >= 0 ? cnt[(size_t)((l - sh) * Cfg::LIMBS + b) * gq + g] : 0u;
            }
        }
        reinterpret_cast<int4 *>(ktop_cur)[q] = kn;
    }
}

// Publish a block's level sums of group g into the absolute-level slot table.
template <int DT, int K>
__device__ __forceinline__ void publish_group(const uint32_t *cnt, int gq, const int64_t (&t)[K], int k, int g,
                                              int32_t *kglob, unsigned long long *slots) {
    constexpr int NS = Fmt<DT>::KMAX + K;
    if (k > 0) atomicMax(&kglob[g], k);
#pragma unroll
    for (int l = 0; l < K; ++l) {
        const int64_t T = t[l] + counters_value<DT, K>(cnt, gq, g, l);
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

// ---- row sources -----------------------------------------------------------
// accumulate_range reads, per input row, one int32 key and NCOL value columns
// and turns them into NV virtual rows (virtual key, value); every virtual row
// is deposited like a row of a single-column GroupBy over the virtual groups.
// R = input rows per thread per tile.  ONES: the last virtual column is the
// constant 1 (COUNT); the fast path deposits its digits -- the same for every
// row under a block-uniform window -- without a digit cascade per row.

// plain GroupBy-SUM of one column
template <int DT>
struct SrcSingle {
    using V = typename Fmt<DT>::V;
    static constexpr int NCOL = 1, NV = 1;
    static constexpr bool ONES = false;  // last virtual column constant 1 (COUNT)
    static constexpr bool KEYLESS = false;  // no key column: every row is group 0
    static constexpr int R = (DT == 1) ? ONCHIP_R64 : ONCHIP_R32;
    const V *col[NCOL];
    int G;
    __device__ __forceinline__ void expand(int32_t key, const V (&c)[NCOL], int32_t (&vk)[NV], V (&vv)[NV]) const {
        vk[0] = key;
        vv[0] = c[0];
    }
};

// Single-array reproducible SUM / dot product (f4 of SURVEY.md 8(f): the
// original setting of the RSum algorithm): no key column,
// every row is group 0; NCOL = 2 multiplies the two columns (one rounding).
template <int DT, int NC>
struct SrcArray {
    using V = typename Fmt<DT>::V;
    static constexpr int NCOL = NC, NV = 1;
    static constexpr bool ONES = false;
    static constexpr bool KEYLESS = true;
    static constexpr int R = (DT == 1) ? ONCHIP_R64 : ONCHIP_R32;
    const V *col[NCOL];
    int G;
    __device__ __forceinline__ void expand(int32_t, const V (&c)[NCOL], int32_t (&vk)[NV], V (&vv)[NV]) const {
        vk[0] = 0;
        vv[0] = NC == 2 ? Fmt<DT>::mul(c[0], c[NC - 1]) : c[0];
    }
};

// The rows of ONE partition (key >> 10 == part) read in place from the
// original columns, as local keys 0..1023 of that partition; every other row
// becomes (its key's low bits, value 0), which deposits nothing and keeps the
// fast path (the partitioned path's heavy-partition offload, k_partition.cu).
// The zero deposits are spread over the groups by the row's own key: sent to
// one group they would pile up on one shared word (14 bank wavefronts per
// warp atomic measured for config 3, vs 3.8 for random groups).
template <int DT>
struct SrcFiltered {
    using V = typename Fmt<DT>::V;
    static constexpr int NCOL = 1, NV = 1;
    static constexpr bool ONES = false;
    static constexpr bool KEYLESS = false;
    static constexpr int R = (DT == 1) ? ONCHIP_R64 : ONCHIP_R32;
    const V *col[NCOL];
    int G;     // groups of the partition (local keys)
    int part;  // partition id
    __device__ __forceinline__ void expand(int32_t key, const V (&c)[NCOL], int32_t (&vk)[NV], V (&vv)[NV]) const {
        const bool in = key >= 0 && (key >> 10) == part;
        vk[0] = in || G == 1024 ? (key & 1023) : (key & 1023) % G;
        vv[0] = in ? c[0] : V(0);
    }
};

// NC columns summed independently plus COUNT: virtual group j * G + g for
// column j, and column NC holds the value 1 for every row (a reproducible sum
// of ones is the exact row count).  Rows with a key outside [0, G) map to
// virtual key -1 (flagged EKEY, never deposited).
template <int DT, int NC>
struct SrcCols {
    using V = typename Fmt<DT>::V;
    static constexpr int NCOL = NC, NV = NC + 1;
    static constexpr bool ONES = true;
    static constexpr bool KEYLESS = false;
    static constexpr int R = ONCHIP_RMULTI;
    const V *col[NCOL];
    int G;
    __device__ __forceinline__ void expand(int32_t key, const V (&c)[NCOL], int32_t (&vk)[NV], V (&vv)[NV]) const {
        const bool ok = (uint32_t)key < (uint32_t)G;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            vk[j] = ok ? key + j * G : -1;
            vv[j] = j < NC ? c[j < NC ? j : 0] : V(1);
        }
    }
};

// The aggregation-heavy query shape of BASELINE config 4 (reading A-15):
// columns (qty, price, disc, tax) -> SUMs of qty, price, disc_price =
// price (x) (1 (-) disc), charge = disc_price (x) (1 (+) tax), each operation
// rounded once (no contraction), plus COUNT.
struct SrcQ1 {
    using V = double;
    static constexpr int NCOL = 4, NV = 5;
    static constexpr bool ONES = true;
    static constexpr bool KEYLESS = false;
    static constexpr int R = ONCHIP_RMULTI;
    const double *col[NCOL];
    int G;
    __device__ __forceinline__ void expand(int32_t key, const double (&c)[NCOL], int32_t (&vk)[NV],
                                           double (&vv)[NV]) const {
        const bool ok = (uint32_t)key < (uint32_t)G;
        const double dp = __dmul_rn(c[1], __dsub_rn(1.0, c[2]));
        vv[0] = c[0];
        vv[1] = c[1];
        vv[2] = dp;
        vv[3] = __dmul_rn(dp, __dadd_rn(1.0, c[3]));
        vv[4] = 1.0;
#pragma unroll
        for (int j = 0; j < NV; ++j) vk[j] = ok ? key + j * G : -1;
    }
};

// Second moments (f2 of SURVEY.md 8(f): AVG / VARIANCE / STDDEV from SUMs,
// PAPER.md:163-174): one column x -> SUM(x), SUM(x (x) x) (one rounding per
// square), COUNT.
template <int DT>
struct SrcMoments {
    using V = typename Fmt<DT>::V;
    static constexpr int NCOL = 1, NV = 3;
    static constexpr bool ONES = true;
    static constexpr bool KEYLESS = false;
    static constexpr int R = ONCHIP_RMULTI;
    const V *col[NCOL];
    int G;
    __device__ __forceinline__ void expand(int32_t key, const V (&c)[NCOL], int32_t (&vk)[NV], V (&vv)[NV]) const {
        const bool ok = (uint32_t)key < (uint32_t)G;
        vv[0] = c[0];
        vv[1] = Fmt<DT>::mul(c[0], c[0]);
        vv[2] = V(1);
#pragma unroll
        for (int j = 0; j < NV; ++j) vk[j] = ok ? key + j * G : -1;
    }
};

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
//
// G is the number of (virtual) groups of the table; SRC (row sources above)
// says how input rows become virtual rows.
template <int DT, int K, bool REGTOT, int MODE, bool TMA = false, class SRC = SrcSingle<DT>>
__device__ __forceinline__ void accumulate_range(const int32_t *__restrict__ keys, const SRC &src, int64_t row0,
                                                 int64_t row1, int32_t G, unsigned char *smem, uint32_t &flags,
                                                 const PubArgs &out) {
    using F = Fmt<DT>;
    using V = typename F::V;
    using Cfg = OnchipCfg<DT, K>;
    constexpr int NCOL = SRC::NCOL, NV = SRC::NV;
    constexpr int TPB = Cfg::TPB, RIN = SRC::R, TILE = TPB * RIN, CW = Cfg::CW;
    constexpr int R = RIN * NV;            // virtual rows per thread per tile
    // fold accounting: a counter of a virtual group receives at most one limb
    // per INPUT row (virtual group j * G + g only gets column j of rows with
    // key g), so the limb headroom is counted in input rows
    constexpr int VTILE = TILE;
    constexpr size_t KB = SRC::KEYLESS ? 0 : 4;      // key bytes per input row
    constexpr size_t ROWB = KB + NCOL * sizeof(V);  // bytes per input row in a ring stage
    static_assert(TILE <= Cfg::LIMIT, "tile larger than limb headroom");
    const int gq = onchip_gq<DT, K>(G, REGTOT);
    const int nq = gq >> 2;  // group quads

    int64_t *tot = reinterpret_cast<int64_t *>(smem);                                   // [GQ][K] (unless REGTOT)
    uint32_t *cnt = reinterpret_cast<uint32_t *>(tot + (REGTOT ? 0 : (size_t)K * gq));  // [CW][GQ]
    int32_t *ktop_cur = reinterpret_cast<int32_t *>(cnt + (size_t)CW * gq);
    int32_t *ktop_next = ktop_cur + gq;
    int32_t *kminmax = ktop_next + gq;  // [0] min, [1] max of ktop_cur over the groups
    const uint32_t cbase = (uint32_t)__cvta_generic_to_shared(cnt);
    const uint32_t wstride = REGTOT ? 4u * Cfg::REG_GQ : 4u * (uint32_t)gq;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    int64_t treg[4][K];  // level sums of groups 4 tid .. 4 tid + 3 (REGTOT)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int l = 0; l < K; ++l) treg[j][l] = 0;
    if (!REGTOT)
        for (int i = tid; i < K * gq; i += TPB) tot[i] = 0;
    for (int i = tid; i < CW * gq; i += TPB) cnt[i] = 0;
    for (int i = tid; i < gq; i += TPB) { ktop_cur[i] = 0; ktop_next[i] = 0; }
    // COUNT column (SRC::ONES): the limbs of 1 under the uniform window,
    // recomputed when the window changes (kminmax[2 .. 2 + 2K))
    uint32_t *climb = reinterpret_cast<uint32_t *>(kminmax + 2);
    auto set_count_limbs = [&](int k) {
        if (SRC::ONES && tid == 0) {
            uint32_t clo[K], chi[K];
            row_limbs<DT, K>(F::pow2(F::m - F::W * k), clo, chi);
#pragma unroll
            for (int l = 0; l < K; ++l) { climb[2 * l] = clo[l]; climb[2 * l + 1] = chi[l]; }
        }
    };
    set_count_limbs(0);
    __shared__ int s_or3[3];
    if (tid < 3) s_or3[tid] = 0;
    BlockOr block_or{s_or3, 0};
    __syncthreads();
    // block-uniform window top: when every group has the same top `kuni`,
    // rows need no per-group lookup (the common case after the first tiles);
    // the fast path's extractors follow it
    int kuni = 0;
    Extractors<DT, K> ex(0);

    // small G: per-lane counter copies (OnchipCfg::LANE_G); their level sums
    // live in shared memory per counter word, rtot[g][w]
    const bool lanerep = REGTOT && G <= ONCHIP_LANEREP;
    int64_t *rtot = reinterpret_cast<int64_t *>(kminmax + 16);
    if (lanerep)
        for (int i = tid; i < Cfg::LANE_G * CW; i += TPB) rtot[i] = 0;
    // the fast path's counter base and per-key stride (bytes)
    const uint32_t fbase = lanerep ? cbase + 4u * lane : cbase;
    const uint32_t kstride = lanerep ? 128u : 4u;

    // lane-copy fold: one thread per (counter word, group) pair sums the 32
    // copies (exact in 32 bits: all copies together hold at most LIMIT rows'
    // worth of limbs) into rtot -- eight 128-bit loads, chunk order rotated by
    // lane so a warp's loads spread over all banks -- then moved groups are
    // demoted (rtot shifts by whole levels; the copies are zero after the fold)
    auto fold_lanes = [&]() {
        for (int p = tid; p < CW * G; p += TPB) {
            const int w = p / G, g = p - w * G;
            uint4 *c = reinterpret_cast<uint4 *>(cnt + (size_t)w * gq + 32 * g);
            uint32_t sum = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int ch = (i + lane) & 7;
                const uint4 v = c[ch];
                sum += v.x + v.y + v.z + v.w;
                c[ch] = make_uint4(0u, 0u, 0u, 0u);
            }
            rtot[g * CW + w] += (int64_t)(int32_t)sum;
        }
        __syncthreads();
        for (int g = tid; g < G; g += TPB) {
            const int sh = ktop_next[g] - ktop_cur[g];
            if (sh != 0) {
                for (int l = K - 1; l >= 0; --l)
                    for (int b = 0; b < Cfg::LIMBS; ++b)
                        rtot[g * CW + l * Cfg::LIMBS + b] = l - sh >= 0 ? rtot[g * CW + (l - sh) * Cfg::LIMBS + b] : 0;
                ktop_cur[g] = ktop_next[g];
            }
        }
    };

    // fold all counters into the level sums, demoting moved groups
    auto fold_all = [&](bool fold) {
        if (lanerep) {
            fold_lanes();
        } else if (REGTOT) {
            fold_quad<DT, K>(cnt, gq, tid, treg, fold, ktop_cur, ktop_next);
        } else {
            for (int q = tid; q < nq; q += TPB) {
                int64_t t[4][K];
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int l = 0; l < K; ++l) t[j][l] = tot[(size_t)(4 * q + j) * K + l];
                fold_quad<DT, K>(cnt, gq, q, t, fold, ktop_cur, ktop_next);
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int l = 0; l < K; ++l) tot[(size_t)(4 * q + j) * K + l] = t[j][l];
            }
        }
    };

    const bool small_g = G <= ONCHIP_SMALLG;
    int since = 0;     // rows' worth of digits in the counters since the last fold
    uint32_t big = 0;  // dynamic fold: bit 31 = an observed counter had |old| >= 2^30
    // dynamic fold (not for lane copies: their folds are cheap, and an atomic
    // that returns its old value costs more than the folds it saves there)
    const bool dyn = ONCHIP_DYNFOLD && !lanerep;

    // a1: coalesced loads (immediate offsets i*TPB from one base pointer),
    // bounds-checked, straight from global memory
    auto expand_row = [&](int i, bool in, int32_t k, const V (&c)[NCOL], int32_t(&key)[R], V(&val)[R]) {
        int32_t vk[NV];
        V vv[NV];
        src.expand(k, c, vk, vv);
#pragma unroll
        for (int j = 0; j < NV; ++j) {  // column-major: virtual row j * RIN + i
            key[j * RIN + i] = in ? vk[j] : -1;
            val[j * RIN + i] = in ? vv[j] : V(0);
        }
    };
    auto load_tile = [&](int64_t b, int32_t(&key)[R], V(&val)[R]) {
        const int rm = (int)min((int64_t)TILE, row1 - b) - tid;
#pragma unroll
        for (int i = 0; i < RIN; ++i) {
            const bool in = i * TPB < rm;
            const int64_t r = b + tid + i * TPB;
            V c[NCOL];
#pragma unroll
            for (int j = 0; j < NCOL; ++j) c[j] = in ? __ldg(src.col[j] + r) : V(0);
            expand_row(i, in, in ? (SRC::KEYLESS ? 0 : __ldg(keys + r)) : -1, c, key, val);
        }
    };
    // TMA-fed variant: full tiles stream through a ring of STAGES shared
    // buffers filled by cp.async.bulk (thread 0 issues, an mbarrier per stage
    // completes on the byte count); tile t lives in stage t % STAGES.  A stage
    // is refilled with tile t + STAGES right after tile t's first barrier, by
    // which point every thread has consumed tile t's rows into registers (the
    // level check reads every loaded register before the barrier), so
    // STAGES - 1 tiles are always in flight while the block works.
    constexpr int S = ONCHIP_STAGES;
    const size_t tbytes = (onchip_table_bytes<DT, K>(G, REGTOT) + 127) & ~(size_t)127;
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)tbytes;  // mbarriers, then tiles
    auto stage_keys = [&](int st) { return ring + 128u + (uint32_t)st * (uint32_t)(TILE * ROWB); };
    auto issue = [&](int64_t t_base, int st) {  // thread 0 only; full tiles only
        const uint32_t bar = ring + 8u * st;
        mbar_expect_tx(bar, (uint32_t)(TILE * ROWB));
        if (!SRC::KEYLESS) tma_load_1d(stage_keys(st), keys + t_base, TILE * 4, bar);
#pragma unroll
        for (int j = 0; j < NCOL; ++j)
            tma_load_1d(stage_keys(st) + (uint32_t)(TILE * (KB + j * sizeof(V))), src.col[j] + t_base,
                        TILE * sizeof(V), bar);
    };
    if (TMA) {
        if (tid == 0) {
            for (int st = 0; st < S; ++st) mbar_init(ring + 8u * st, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0)
            for (int st = 0; st < S; ++st)
                if (row0 + (int64_t)(st + 1) * TILE <= row1) issue(row0 + (int64_t)st * TILE, st);
    }

    int tile = 0;
    for (int64_t base = row0; base < row1; base += TILE, ++tile) {
        const int rem = (int)min((int64_t)TILE, row1 - base) - tid;  // rows i*TPB < rem exist
        int32_t key[R];
        V val[R];
        int kc[R];
        if (TMA && base + TILE <= row1) {
            const int st = tile % S;
            mbar_wait(ring + 8u * st, (uint32_t)((tile / S) & 1));
            const int32_t *sk = reinterpret_cast<const int32_t *>(smem + tbytes + 128 + (size_t)st * TILE * ROWB);
            const V *sv = reinterpret_cast<const V *>(reinterpret_cast<const unsigned char *>(sk) + TILE * KB);
#pragma unroll
            for (int i = 0; i < RIN; ++i) {
                V c[NCOL];
#pragma unroll
                for (int j = 0; j < NCOL; ++j) c[j] = sv[j * TILE + tid + i * TPB];
                expand_row(i, true, SRC::KEYLESS ? 0 : sk[tid + i * TPB], c, key, val);
            }
        } else {
            load_tile(base, key, val);
        }
        // refill this tile's stage (right after the tile's first barrier)
        auto refill = [&]() {
            if (TMA && tid == 0 && base + (int64_t)(S + 1) * TILE <= row1) {
                fence_proxy_async_smem();
                issue(base + (int64_t)S * TILE, tile % S);
            }
        };
        // Fast path: when the block has a uniform window top kuni and every row
        // of this full tile has a valid key and needs no level shift, the tile
        // is deposited without per-row checks.  One barrier decides it for the
        // whole block (and orders the previous tile's deposits before a fold).
        if (ONCHIP_FAST && !small_g) {
            // bit 0: this thread's rows need the generic code; bit 1: a counter
            // neared 2^30 (dynamic fold).  The row checks run whatever bit 1
            // says: a pending fold must not let a bad row through the fast path.
            int slow = kuni < 0 || rem < TILE - tid;
            if (!slow) {
                // k*(b) <= kuni  <=>  |b| < 2^(W kuni + W - 1 - m): compare the
                // magnitude bits (sign shifted out); NaN/Inf fail it too
                const uint32_t lim = (uint32_t)(F::W * kuni + F::W - 1 - F::m + F::BIAS) << (F::m % 32 + 1);
                uint32_t hwmax = 0, kmax = 0;
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    uint32_t hw;
                    if (DT == 1) hw = (uint32_t)__double2hiint((double)val[i]) << 1;
                    else hw = __float_as_uint((float)val[i]) << 1;
                    hwmax = max(hwmax, hw);
                    kmax = max(kmax, (uint32_t)key[i]);
                }
                slow = (hwmax >= lim) | (kmax >= (uint32_t)G);
            }
            slow |= (int)(big >> 31) << 1;
            const int any_flags = block_or(slow);
            const int any_slow = any_flags & 1;
            refill();
            if (!any_slow) {
                // static cadence: fold every LIMIT rows.  Dynamic (ONCHIP_DYNFOLD,
                // every deposit returns the counter's old value): fold when a
                // counter was seen at |old| >= 2^30 in the previous tile; with
                // at most TILE deposits per counter per tile a counter then
                // stays below 2^30 + (TILE + 1) 2^19 < 2^31
                const bool fold_now = dyn ? (any_flags & 2) != 0 : since + VTILE > Cfg::LIMIT;
                if (fold_now) {
                    fold_all(true);
                    since = 0;
                    big = 0;
                    __syncthreads();
                }
                if (!dyn) since += VTILE;
                constexpr int RD = SRC::ONES ? R - RIN : R;  // virtual rows with a digit cascade
                constexpr int NB = ONCHIP_NB < RD ? ONCHIP_NB : RD;
#pragma unroll
                for (int i0 = 0; i0 < RD; i0 += NB) {
                    constexpr int NL = RD % NB ? RD % NB : NB;
                    if (dyn) {
                        if (i0 + NB <= RD)
                            deposit_batch<DT, K, NB, true>(fbase, kstride, wstride, key + i0, val + i0, ex, big);
                        else
                            deposit_batch<DT, K, NL, true>(fbase, kstride, wstride, key + i0, val + i0, ex, big);
                    } else {
                        if (i0 + NB <= RD)
                            deposit_batch<DT, K, NB, false>(fbase, kstride, wstride, key + i0, val + i0, ex, big);
                        else
                            deposit_batch<DT, K, NL, false>(fbase, kstride, wstride, key + i0, val + i0, ex, big);
                    }
                }
                if (SRC::ONES) {
                    // COUNT column: the limbs of 1 under the window kuni
#pragma unroll
                    for (int l = 0; l < K; ++l) {
#pragma unroll
                        for (int h = 0; h < Cfg::LIMBS; ++h) {
                            const uint32_t c = climb[2 * l + (Cfg::LIMBS == 2 ? h : 0)];
                            if (c != 0u) {
                                const uint32_t off = (uint32_t)(Cfg::LIMBS * l + h) * wstride;
#pragma unroll
                                for (int i = 0; i < RIN; ++i) {  // fast path: every key is valid
                                    if (dyn) red_shared_obs(fbase + kstride * (uint32_t)key[R - RIN + i] + off, c, big);
                                    else red_shared(fbase + kstride * (uint32_t)key[R - RIN + i] + off, c);
                                }
                            }
                        }
                    }
                }
                continue;
            }
        }
        // a2: window tops; raise ktop_next of the row's group where needed
        int changed = 0;
        if (kuni >= 0) {
#pragma unroll
            for (int i = 0; i < R; ++i) {
                int ks;
                const int k = check_row<DT>(key[i], val[i], (i % RIN) * TPB < rem, G, flags, ks);
                if (k >= 0 && ks > kuni) { atomicMax(&ktop_next[k], ks); changed = 1; }
                key[i] = k;
                kc[i] = kuni;
            }
        } else {
#pragma unroll
            for (int i = 0; i < R; ++i) {
                int ks;
                const int k = check_row<DT>(key[i], val[i], (i % RIN) * TPB < rem, G, flags, ks);
                const int cur = k >= 0 ? ktop_cur[k] : 0;
                if (k >= 0 && ks > cur) { atomicMax(&ktop_next[k], ks); changed = 1; }
                key[i] = k;
                kc[i] = cur;
            }
        }
        // dynamic mode: every deposit is observed; fold when a counter was
        // seen at |old| >= 2^30 (bit 1 of the barrier's OR)
        const int any_flags = block_or(changed | (int)(big >> 31) << 1);  // + previous tile done
        const int any = any_flags & 1;
        const bool fold = dyn ? (any_flags & 2) != 0 : since + VTILE > Cfg::LIMIT;
        if (!(ONCHIP_FAST && !small_g)) refill();
        if (any || fold) {
            // fold counters into the level sums and demote moved groups
            fold_all(fold);
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
            if (fold) {
                since = 0;
                big = 0;
            }
            if (any) {
                kuni = kminmax[0] == kminmax[1] ? kminmax[1] : -1;
                if (kuni >= 0) {
                    ex = Extractors<DT, K>(kuni);
                    set_count_limbs(kuni);  // ordered before use by the next tile's barrier
                }
#pragma unroll
                for (int i = 0; i < R; ++i)
                    if (key[i] >= 0) kc[i] = ktop_cur[key[i]];
            }
        }
        since += VTILE;

        // a3 + a4: digits under the group's current top, 32-bit shared atomics
        if (small_g) {
#pragma unroll
            for (int i = 0; i < R; ++i)
                deposit_row<DT, K, true>(cnt, gq, key[i], F::mul(val[i], F::pow2(F::m - F::W * kc[i])), lane);
        } else if (lanerep) {
#pragma unroll
            for (int i = 0; i < R; ++i)
                deposit_row<DT, K, false>(cnt + lane, gq, key[i] >= 0 ? 32 * key[i] : -1,
                                          F::mul(val[i], F::pow2(F::m - F::W * kc[i])), lane);
        } else if (dyn) {
#pragma unroll
            for (int i = 0; i < R; ++i)
                deposit_row<DT, K, false, true>(cnt, gq, key[i], F::mul(val[i], F::pow2(F::m - F::W * kc[i])), lane,
                                                &big);
        } else if (kuni >= 0) {
            const V scale = F::pow2(F::m - F::W * kuni);
#pragma unroll
            for (int i = 0; i < R; ++i) deposit_row<DT, K, false>(cnt, gq, key[i], F::mul(val[i], scale), lane);
        } else {
#pragma unroll
            for (int i = 0; i < R; ++i)
                deposit_row<DT, K, false>(cnt, gq, key[i], F::mul(val[i], F::pow2(F::m - F::W * kc[i])), lane);
        }
    }

    // flush: publish the block's table (level sums + unfolded counters;
    // replicated counters are folded first)
    __syncthreads();
    if (lanerep) {
        fold_lanes();
        __syncthreads();
    }
    auto pub = [&](int g, const int64_t(&t)[K]) {
        if (MODE == 0) {
            publish_group<DT, K>(cnt, gq, t, ktop_cur[g], g, out.kglob, out.slots);
        } else {
            out.pk[g] = ktop_cur[g];
#pragma unroll
            for (int l = 0; l < K; ++l) out.pT[(size_t)g * K + l] = t[l] + counters_value<DT, K>(cnt, gq, g, l);
        }
    };
    if (lanerep) {
        for (int g = tid; g < G; g += TPB) {
            int64_t t[K];
#pragma unroll
            for (int l = 0; l < K; ++l)
                t[l] = Cfg::LIMBS == 2 ? rtot[g * CW + 2 * l] + rtot[g * CW + 2 * l + 1] * (int64_t)(1 << 20)
                                       : rtot[g * CW + l];
            pub(g, t);  // the lane copies are all zero after the final fold
        }
    } else if (REGTOT) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (4 * tid + j < G) pub(4 * tid + j, treg[j]);
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
