// k_lean.cu -- the fused multi-column GroupBy for a handful of groups
// (BASELINE config 4's shape: 4 groups, 4 SUMs + COUNT), built for issue
// efficiency.
//
// The on-chip kernel handles any group count with block-wide tables, a tile
// barrier per TMA stage, per-tile window checks and one warp vote per counter
// position; for config 4 (two input rows per thread per tile, 20 virtual
// groups) that machinery costs ~290 warp instructions per 32 rows and the
// kernel is issue-bound at half the HBM roofline.  Here:
//  * every WARP owns a private counter table with one copy per lane (bank =
//    lane: conflict-free 32-bit shared atomics, no block barriers), folded by
//    the warp itself (__syncwarp) every FOLD_IT iterations into per-warp int64
//    level sums;
//  * rows come straight from HBM in 16-byte vectors (4 rows per thread per
//    iteration: one int4 of keys, two V-pairs per column);
//  * all of a block's values must sit at ONE lattice window k0 (the window of
//    the block's first value): k*(b) == k0 for every value, checked with one
//    magnitude range test per value; then every (group, column) the block
//    touches has top exactly k0, the extractors are fixed, and no level shift
//    or per-row window bookkeeping exists.  A block that meets any other value
//    (another window, a zero when k0 > 0, NaN/Inf, a key outside [0, G)) drops
//    its tables and runs the on-chip kernel's generic code (accumulate_range)
//    over its whole row range instead -- the result and the status bits never
//    depend on which code a block ran;
//  * COUNT (the last virtual column) is published from exact per-group row
//    counts at level 1 (digit 2^(m - W) per row, reading A-16).
// Digits and limbs are those of the on-chip fast path (Extractors,
// deposit_batch in onchip_core.cuh): identical integers, so identical bits.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"

#include <algorithm>

namespace repro {

namespace {

bool lean_disabled() { return onchip_variant() != 0; }  // variants 1-3 force the on-chip kernel

#ifndef LEAN_PIPE
#define LEAN_PIPE 1  // prefetch the next quad of rows while depositing this one
#endif
#ifndef LEAN_L2PF
#define LEAN_L2PF 0  // > 0: lane 0 of each warp bulk-prefetches its rows that many steps ahead into L2 (measured slower: config 4 7.9 -> 9.2 ms)
#endif
#ifndef LEAN_MINB
#define LEAN_MINB 1  // resident blocks per SM the register budget is sized for
#endif
__device__ __forceinline__ void l2_prefetch_lean(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}
constexpr int LEAN_TPB = 256;  // = OnchipCfg::TPB (the fallback runs accumulate_range)
constexpr int LEAN_GL = 4;     // groups handled (multi-column sources)
constexpr int LEAN_GL1 = 16;   // groups handled (single column)
constexpr int LEAN_U = 4;      // rows per thread per iteration
// a lane copy takes <= 1 limb per row of its lane; the 32 copies of a counter
// are summed in 32 bits, so a fold is due every 4095 / 32 rows per lane

template <int DT>
struct LeanVec;
template <>
struct LeanVec<1> {  // 4 doubles = two 16-byte loads
    __device__ __forceinline__ static void load(const double *p, double (&o)[4]) {
        const double2 a = __ldcs(reinterpret_cast<const double2 *>(p));
        const double2 b = __ldcs(reinterpret_cast<const double2 *>(p) + 1);
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    }
};
template <>
struct LeanVec<0> {  // 4 floats = one 16-byte load
    __device__ __forceinline__ static void load(const float *p, float (&o)[4]) {
        const float4 a = __ldcs(reinterpret_cast<const float4 *>(p));
        o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    }
};

template <int DT, int K, class SRC, int GL>
struct LeanGeom {
    static constexpr int NV = SRC::NV;
    static constexpr int ND = SRC::ONES ? NV - 1 : NV;  // virtual columns with digits
    static constexpr int CW = K * Fmt<DT>::LIMBS;        // counter words per virtual group
    static constexpr int NPOS = ND * GL * CW;            // counter positions per warp (x 32 lanes)
    static constexpr int WORDS = (NPOS + GL) * 32;       // + per-group row counts
    static constexpr size_t WARP_BYTES = 4 * (size_t)WORDS + 8 * (size_t)(NPOS + GL);  // + int64 sums
    static constexpr size_t BYTES = WARP_BYTES * (LEAN_TPB / 32);
    static_assert(ND * GL <= 32, "one bit per (column, group) in the window masks");
};

template <int DT, int K, class SRC, int GL>
__global__ void __launch_bounds__(LEAN_TPB, LEAN_MINB)
k_lean_multi(const int32_t *__restrict__ keys, const SRC src, int64_t n, int32_t G, int64_t chunk,
             int32_t *__restrict__ kglob, unsigned long long *__restrict__ slots, uint32_t *__restrict__ status) {
    using F = Fmt<DT>;
    using V = typename F::V;
    using Geo = LeanGeom<DT, K, SRC, GL>;
    using Cfg = OnchipCfg<DT, K>;
    constexpr int NV = Geo::NV, ND = Geo::ND, CW = Geo::CW, NPOS = Geo::NPOS;
    constexpr int NS = F::KMAX + K;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_bad, s_k0;
    __shared__ uint32_t s_present, s_seen;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t row0 = (int64_t)blockIdx.x * chunk;
    const int64_t row1 = min(n, row0 + chunk);
    if (row0 >= row1) return;

    // this warp's table: counters [NPOS][32] (position p = (j * GL + g) * CW + w),
    // COUNT copies [GL][32], then int64 sums [NPOS + GL]
    uint32_t *wt = reinterpret_cast<uint32_t *>(smem + (size_t)warp * Geo::WARP_BYTES);
    int64_t *wsum = reinterpret_cast<int64_t *>(wt + Geo::WORDS);
    for (int i = lane; i < Geo::WORDS; i += 32) wt[i] = 0;
    for (int i = lane; i < NPOS + GL; i += 32) wsum[i] = 0;
    if (tid == 0) {
        s_bad = 0;
        s_k0 = 0;
        s_present = 0;
        s_seen = 0;
    }
    __syncthreads();
    {  // the block's window k0: the largest k* among the first LEAN_TPB rows
        const int64_t r = row0 + tid;
        if (r < row1) {
            V c[SRC::NCOL];
#pragma unroll
            for (int j = 0; j < SRC::NCOL; ++j) c[j] = src.col[j][r];
            int32_t vk[NV];
            V vv[NV];
            src.expand(0, c, vk, vv);
            int km = 0;
#pragma unroll
            for (int j = 0; j < ND; ++j) {
                uint32_t f = 0;
                km = max(km, kstar_of<DT>(vv[j], f));
            }
            km = __reduce_max_sync(__activemask(), km);  // active lanes are a prefix: lane 0 is one
            if (lane == 0) atomicMax(&s_k0, km);
        }
    }
    __syncthreads();
    const int k0 = s_k0;
    // k*(b) <= k0  <=>  |b| < hi on the magnitude bits (NaN/Inf fail it);
    // k*(b) == k0  <=>  also |b| >= lo (k0 > 0), tracked per (column, group)
    const uint32_t sh = DT == 1 ? 20 : 23;
    const uint32_t hi_b = (uint32_t)(F::W * k0 + F::W - 1 - F::m + F::BIAS) << sh;
    const uint32_t lo_b = k0 == 0 ? 0u : (uint32_t)(F::W * (k0 - 1) + F::W - 1 - F::m + F::BIAS) << sh;
    const Extractors<DT, K> ex(k0);
    const uint32_t tbase = (uint32_t)__cvta_generic_to_shared(wt) + 4u * (uint32_t)lane;
    const uint32_t cbase = tbase + 4u * 32u * (uint32_t)NPOS;  // COUNT copies

    // fold: sum the 32 lane copies of every position into the warp's int64
    // sums and clear them.  The counters hold RAW limbs (see take): the sum
    // of a position is corrected by (rows of its group since the last fold) x
    // (the limb's constant bias), mod 2^32 -- exact, since the true sum of at
    // most 32 x 4Q x FOLD_IT <= 4095 balanced limbs fits an int32.
    auto copies_sum = [&](int p) {
        uint4 *c = reinterpret_cast<uint4 *>(wt + (size_t)p * 32);
        uint32_t s = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int ch = (i + lane) & 7;
            const uint4 v = c[ch];
            s += v.x + v.y + v.z + v.w;
            c[ch] = make_uint4(0u, 0u, 0u, 0u);
        }
        return s;
    };
    auto fold = [&]() {
        __syncwarp();
        uint32_t ng = 0;
        if (lane < GL) {
            ng = copies_sum(NPOS + lane);
            wsum[NPOS + lane] += (int64_t)ng;
        }
        for (int p0 = 0; p0 < NPOS; p0 += 32) {  // warp-uniform trip count (shuffles below)
            const int p = p0 + lane;
            const int g = (p / CW) % GL, w = p % CW;
            const uint32_t nsel = __shfl_sync(0xffffffffu, ng, g);  // rows of group g since the last fold
            if (p >= NPOS) continue;
            uint32_t bias;
            if (DT == 1) {
                bias = (w & 1) ? 0x80000000u : 0x80000u;  // hi: exponent field of E_l; lo: the 2^19 offset
            } else {
                const int ue = F::W * (k0 - w) - F::m;  // binary32: one limb per level, bias = bits(E_l)
                bias = ((uint32_t)(ue + F::m + F::BIAS) << 23) | (1u << 22);
            }
            const uint32_t s = copies_sum(p) - bias * nsel;
            wsum[p] += (int64_t)(int32_t)s;
        }
        __syncwarp();
    };

    // deposit one row: digits of the ND virtual values under k0 as RAW limbs
    // (the balanced limbs of the on-chip kernel plus a constant per limb,
    // removed at the fold), one conflict-free atomic per limb, +1 on the
    // group's COUNT copy.
    // Position (j * GL + g) * CW + w sits at byte 128 * position of the table.
    uint32_t present = 0, seen = 0;  // groups with rows; (column, group) with a value at k0
    auto take = [&](int32_t key, const V (&c)[SRC::NCOL], bool &bad) {
        int32_t vk[NV];
        V vv[NV];
        src.expand(key, c, vk, vv);
        bad |= (uint32_t)key >= (uint32_t)G;
        const uint32_t g = (uint32_t)key & (GL - 1);
        const uint32_t kb = tbase + 128u * CW * g;
        const uint32_t gbit = 1u << g;
        present |= gbit;
#pragma unroll
        for (int j = 0; j < ND; ++j) {
            const uint32_t a = (DT == 1 ? (uint32_t)__double2hiint((double)vv[j]) : __float_as_uint((float)vv[j])) &
                               0x7FFFFFFFu;
            bad |= a >= hi_b;
            seen |= a >= lo_b ? gbit << (j * GL) : 0u;
            V r = vv[j];
#pragma unroll
            for (int l = 0; l < K; ++l) {
                uint32_t lo, hi = 0;
                if (DT == 1) {
                    const double x = __hiloint2double(__double2hiint((double)r), __double2loint((double)r) | 1);
                    const double t = __dadd_rn(x, (double)ex.e[l]);
                    const uint32_t tlo = (uint32_t)__double2loint(t), thi = (uint32_t)__double2hiint(t);
                    lo = tlo & 0xFFFFFu;                 // raw: balanced limb + 2^19
                    hi = __funnelshift_r(tlo, thi, 20);  // raw: balanced limb + 2^31 (ex.eb[l])
                    if (l + 1 < K) r = (V)__dsub_rn((double)r, __dsub_rn(t, (double)ex.e[l]));
                } else {
                    const float x = __uint_as_float(__float_as_uint((float)r) | 1u);
                    const float t = __fadd_rn(x, (float)ex.e[l]);
                    lo = __float_as_uint(t);  // raw: digit + bits(E_l)
                    if (l + 1 < K) r = (V)__fsub_rn((float)r, __fsub_rn(t, (float)ex.e[l]));
                }
                const uint32_t off = 128u * (uint32_t)(j * GL * CW + l * Cfg::LIMBS);
                red_shared(kb + off, lo);
                if (Cfg::LIMBS == 2) red_shared(kb + off + 128u, hi);
            }
        }
        red_shared(cbase + 128u * g, 1u);
    };

    bool bad = false;
    const int64_t nq = (row1 - row0) / LEAN_U;  // whole quads (row0 % 4 == 0)
    // Q quads per thread per step (interleaved: quad q0 + i * TPB + tid, so
    // every 16-byte load instruction of a warp is contiguous); Q grows as the
    // row gets narrower, keeping ~128-192 bytes per lane in flight
    constexpr int Q = SRC::NCOL == 1 ? 4 : SRC::NCOL == 2 ? 2 : 1;
    constexpr int FOLD_IT = 4095 / 32 / (LEAN_U * Q);  // a lane copy takes <= 4Q rows per step
    int it = 0;
    // software pipeline: the next step's loads are in flight while this one
    // is deposited
    int4 kk[Q];
    V cv[Q][SRC::NCOL][4];
    auto load_step = [&](int64_t q0) {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int64_t q = q0 + i * LEAN_TPB + tid;
            if (q < nq) {
                const int64_t r = row0 + q * LEAN_U;
                kk[i] = __ldcs(reinterpret_cast<const int4 *>(keys + r));
#pragma unroll
                for (int j = 0; j < SRC::NCOL; ++j) LeanVec<DT>::load(src.col[j] + r, cv[i][j]);
            }
        }
    };
    if (LEAN_PIPE) load_step(0);
    for (int64_t q0 = 0; q0 < nq; q0 += Q * LEAN_TPB) {  // warp-uniform trip count
        if (!LEAN_PIPE) load_step(q0);
        int4 k_cur[Q];
        V c_cur[Q][SRC::NCOL][4];
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            k_cur[i] = kk[i];
#pragma unroll
            for (int j = 0; j < SRC::NCOL; ++j)
#pragma unroll
                for (int u = 0; u < 4; ++u) c_cur[i][j][u] = cv[i][j][u];
        }
        if (LEAN_PIPE) load_step(q0 + Q * LEAN_TPB);
        if (LEAN_L2PF && lane == 0) {  // the warp's rows LEAN_L2PF steps ahead, into L2 (no registers)
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                const int64_t qp = q0 + (int64_t)(LEAN_L2PF * Q + i) * LEAN_TPB + tid;  // (lane 0: the warp's first quad)
                if (qp + 32 <= nq) {
                    const int64_t r = row0 + qp * LEAN_U;
                    l2_prefetch_lean(keys + r, 128 * 4);
#pragma unroll
                    for (int j = 0; j < SRC::NCOL; ++j) l2_prefetch_lean(src.col[j] + r, 128 * (uint32_t)sizeof(V));
                }
            }
        }
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            if (q0 + i * LEAN_TPB + tid < nq) {
                const int32_t ks[4] = {k_cur[i].x, k_cur[i].y, k_cur[i].z, k_cur[i].w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    V c[SRC::NCOL];
#pragma unroll
                    for (int j = 0; j < SRC::NCOL; ++j) c[j] = c_cur[i][j][u];
                    take(ks[u], c, bad);
                }
            }
        }
        // a value outside the lean path anywhere in the block: stop (the
        // decision is warp-uniform; the block falls back below)
        if (__any_sync(0xffffffffu, bad || *(volatile int *)&s_bad)) {
            if (lane == 0) atomicOr(&s_bad, 1);
            bad = true;
            break;
        }
        if (++it == FOLD_IT) {
            fold();
            it = 0;
        }
    }
    // the last < 4 rows of the range (scalar, one per thread)
    if (!bad) {
        const int64_t r = row0 + nq * LEAN_U + tid;
        if (r < row1) {
            V c[SRC::NCOL];
#pragma unroll
            for (int j = 0; j < SRC::NCOL; ++j) c[j] = src.col[j][r];
            take(keys[r], c, bad);
        }
        if (bad) atomicOr(&s_bad, 1);
    }
    present = __reduce_or_sync(0xffffffffu, present);
    seen = __reduce_or_sync(0xffffffffu, seen);
    if (lane == 0) {
        atomicOr(&s_present, present);
        atomicOr(&s_seen, seen);
    }
    __syncthreads();
    if (tid == 0) {
        // every (column, group) the block touched needs a value AT k0, or its
        // top in this block is lower and the levels under k0 - K + 1 that were
        // dropped may be needed: such a block takes the generic code
#pragma unroll
        for (int j = 0; j < ND; ++j)
            if (s_present & ~(s_seen >> (j * GL)) & (GL == 32 ? 0xffffffffu : (1u << GL) - 1u)) s_bad = 1;
    }
    __syncthreads();

    if (s_bad) {
        // generic on-chip code over the whole row range (register loads); the
        // lean tables are abandoned (accumulate_range re-initialises smem)
        uint32_t flags = 0;
        PubArgs out{kglob, slots, nullptr, nullptr};
        accumulate_range<DT, K, true, 0, false, SRC>(keys, src, row0, row1, G * NV, smem, flags, out);
        flags = __reduce_or_sync(0xffffffffu, flags);
        if (lane == 0 && flags) atomicOr(status, flags);
        return;
    }
    fold();
    __syncthreads();

    // publish: one thread per (virtual column j, group g, level l), plus COUNT;
    // the warps' sums are added here
    for (int p = tid; p < ND * G * K + G; p += LEAN_TPB) {
        if (p < ND * G * K) {
            const int j = p / (G * K), g = (p / K) % G, l = p % K;
            int64_t s = 0, c = 0;
            const int pos = (j * GL + g) * CW + l * Cfg::LIMBS;
            for (int w = 0; w < LEAN_TPB / 32; ++w) {
                const int64_t *ws = reinterpret_cast<const int64_t *>(
                    reinterpret_cast<const uint32_t *>(smem + (size_t)w * Geo::WARP_BYTES) + Geo::WORDS);
                s += ws[pos] + (Cfg::LIMBS == 2 ? ws[pos + 1] * (int64_t)(1 << 20) : 0);
                c += ws[NPOS + g];
            }
            if (c == 0) continue;  // the block has no row of this group
            const int vg = j * G + g;
            if (l == 0 && k0 > 0) atomicMax(&kglob[vg], k0);
            if (s != 0) {
                unsigned long long *q = slots + ((size_t)vg * NS + (k0 - l + K - 1)) * 2;
                atomicAdd(q, (unsigned long long)(s & 0xFFFFFFFFll));
                atomicAdd(q + 1, (unsigned long long)(s >> 32));
            }
        } else if (SRC::ONES) {
            // COUNT: window top k*(1) = 1, level-1 digit 2^(m - W) per row
            const int g = p - ND * G * K;
            int64_t c = 0;
            for (int w = 0; w < LEAN_TPB / 32; ++w)
                c += reinterpret_cast<const int64_t *>(
                    reinterpret_cast<const uint32_t *>(smem + (size_t)w * Geo::WARP_BYTES) + Geo::WORDS)[NPOS + g];
            if (c == 0) continue;
            const int vg = ND * G + g;
            atomicMax(&kglob[vg], 1);
            const int64_t s = c << (F::m - F::W);
            unsigned long long *q = slots + ((size_t)vg * NS + (1 + K - 1)) * 2;
            atomicAdd(q, (unsigned long long)(s & 0xFFFFFFFFll));
            atomicAdd(q + 1, (unsigned long long)(s >> 32));
        }
    }
}

template <int DT, int K, class SRC, int GL>
int launch_lean_t(const int32_t *keys, const SRC &src, int64_t n, int32_t G, int32_t *kglob,
                  unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
    using Geo = LeanGeom<DT, K, SRC, GL>;
    if (G > GL) return 1;
    const int32_t Gv = G * SRC::NV;
    // the lean tables, or the fallback's shared table (register level sums,
    // register loads) -- whichever is larger (the two are never live together)
    const size_t fb = (onchip_table_bytes<DT, K>(Gv, true) + 127) & ~(size_t)127;
    const size_t smem = std::max(fb, Geo::BYTES);
    auto kern = k_lean_multi<DT, K, SRC, GL>;
    if (smem > (size_t)device_props().smem_optin) return 1;
    static thread_local size_t configured = 0;
    if (configured < smem) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return -2;
        configured = smem;
    }
    if (n == 0) return 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LEAN_TPB, smem);
    if (per_sm < 1) return 1;
    int64_t grid = (int64_t)per_sm * device_props().sms;
    // <= 2^23 rows per block (the fallback's int64 level sums)
    const int64_t min_grid = (n + (1ll << 23) - 1) >> 23;
    if (grid < min_grid) grid = min_grid;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = (chunk + 1023) / 1024 * 1024;
    if (chunk > (1ll << 23)) chunk = 1ll << 23;
    grid = (n + chunk - 1) / chunk;
    kern<<<(unsigned)grid, LEAN_TPB, smem, st>>>(keys, src, n, G, chunk, kglob, slots, status);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace

// whether launch_lean_multi takes this call (for the per-kernel timing label)
bool lean_multi_applies(int DT, int proj, int ncols, const int32_t *keys, const void *const *cols, int32_t G) {
    if (G > LEAN_GL || lean_disabled()) return false;
    const bool shape = proj == 1 ? (DT == 1 && ncols == 4) : proj == 2 ? ncols == 1
                                                                          : (ncols == 1 || ncols == 2 || ncols == 4);
    if (!shape) return false;
    uintptr_t al = (uintptr_t)keys;
    for (int j = 0; j < ncols; ++j) al |= (uintptr_t)cols[j];
    return (al & 15) == 0;
}

// 0 = launched, 1 = shape not handled here (the caller uses the on-chip
// kernel), < 0 = error.  Needs 16-byte aligned key and value columns, G <= 4.
int launch_lean_multi(int DT, int K, int proj, int ncols, const int32_t *keys, const void *const *cols, int64_t n,
                      int32_t G, int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                      int *launches) {
#define LEAN_K(dt, SRCT)                                                                                       \
    do {                                                                                                       \
        SRCT src;                                                                                              \
        for (int j = 0; j < SRCT::NCOL; ++j) src.col[j] = (const typename Fmt<dt>::V *)cols[j];               \
        src.G = G;                                                                                             \
        switch (K) {                                                                                           \
            case 1: return launch_lean_t<dt, 1, SRCT, LEAN_GL>(keys, src, n, G, kglob, slots, status, st, launches); \
            case 2: return launch_lean_t<dt, 2, SRCT, LEAN_GL>(keys, src, n, G, kglob, slots, status, st, launches); \
            case 3: return launch_lean_t<dt, 3, SRCT, LEAN_GL>(keys, src, n, G, kglob, slots, status, st, launches); \
            case 4: return launch_lean_t<dt, 4, SRCT, LEAN_GL>(keys, src, n, G, kglob, slots, status, st, launches); \
        }                                                                                                      \
        return 1;                                                                                              \
    } while (0)
    if (!lean_multi_applies(DT, proj, ncols, keys, cols, G)) return 1;
    using C64_1 = SrcCols<1, 1>;
    using C64_2 = SrcCols<1, 2>;
    using C64_4 = SrcCols<1, 4>;
    using C32_1 = SrcCols<0, 1>;
    using C32_2 = SrcCols<0, 2>;
    using C32_4 = SrcCols<0, 4>;
    using M64 = SrcMoments<1>;
    using M32 = SrcMoments<0>;
    if (proj == 1) LEAN_K(1, SrcQ1);
    if (proj == 2) {
        if (DT == 1) LEAN_K(1, M64);
        LEAN_K(0, M32);
    }
    if (DT == 1) {
        if (ncols == 1) LEAN_K(1, C64_1);
        if (ncols == 2) LEAN_K(1, C64_2);
        LEAN_K(1, C64_4);
    }
    if (ncols == 1) LEAN_K(0, C32_1);
    if (ncols == 2) LEAN_K(0, C32_2);
    LEAN_K(0, C32_4);
#undef LEAN_K
}

// Single-column GroupBy with at most LEAN_GL1 groups (16-byte aligned
// columns): 0 = launched, 1 = not handled here.
bool lean_single_applies(const int32_t *keys, const void *vals, int32_t G) {
    return G <= LEAN_GL1 && !lean_disabled() && (((uintptr_t)keys | (uintptr_t)vals) & 15) == 0;
}

int launch_lean_single(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t *kglob,
                       unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
    if (!lean_single_applies(keys, vals, G)) return 1;
#define LEAN_S(dt)                                                                                               \
    do {                                                                                                         \
        SrcSingle<dt> src;                                                                                       \
        src.col[0] = (const typename Fmt<dt>::V *)vals;                                                          \
        src.G = G;                                                                                               \
        switch (K) {                                                                                             \
            case 1: return launch_lean_t<dt, 1, SrcSingle<dt>, LEAN_GL1>(keys, src, n, G, kglob, slots, status, st, launches); \
            case 2: return launch_lean_t<dt, 2, SrcSingle<dt>, LEAN_GL1>(keys, src, n, G, kglob, slots, status, st, launches); \
            case 3: return launch_lean_t<dt, 3, SrcSingle<dt>, LEAN_GL1>(keys, src, n, G, kglob, slots, status, st, launches); \
            case 4: return launch_lean_t<dt, 4, SrcSingle<dt>, LEAN_GL1>(keys, src, n, G, kglob, slots, status, st, launches); \
        }                                                                                                        \
        return 1;                                                                                                \
    } while (0)
    if (DT == 1) LEAN_S(1);
    LEAN_S(0);
#undef LEAN_S
}

}  // namespace repro
