// table_core.cuh -- the block-wide limb-counter table behind k_table (the
// on-chip GroupBy, k_table.cu) and the partitioned path's sweep and
// per-partition accumulation (k_sweep.cu).  See k_table.cu for the design:
// word-major 32-bit limb counters in shared memory, one window top per
// group, every level sum published into the ABSOLUTE-LEVEL slot table
// (counter drains at |old| >= 2^29, demotions, the final flush), a
// block-synchronous mode until every group shares one window top and a
// barrier-free streaming mode after it.
#pragma once

#include "common.cuh"
#include "onchip_core.cuh"

namespace repro {

constexpr uint32_t TAB_DRAIN_BIAS = 0x20000000u;  // |old| >= 2^29  <=>  (old + 2^29) has bit 30 or 31
constexpr uint32_t TAB_DRAIN_MASK = 0xC0000000u;
constexpr int TAB_MM = 64;  // shared control words of a Table: lists, tops, rows per k* (first tile), NTOP
constexpr int TAB_HMAX = 32;
// rows that are not deposited add zeros into a SINK column of their own lane
// (G + lane: bank = lane), so that they never pile up on one shared word
constexpr int TAB_SINKS = 32;
#ifndef TAB_DEBUG
#define TAB_DEBUG 0  // count the calls per table mode (repro_debug_table_modes; debug builds only)
#endif
#ifndef TAB_BAND_CHECK
#define TAB_BAND_CHECK 4  // band-mode calls before the first check for the switch to the uniform mode
#endif
#ifndef TAB_BAND_CHECK_MAX
#define TAB_BAND_CHECK_MAX 1024  // the interval doubles after every check that fails (skewed keys: never)
#endif
#ifndef TAB_VOTE_LO
#define TAB_VOTE_LO 1  // vote on the low limbs of binary64 digits too (skip a position the warp leaves at zero)
#endif  // heavy groups with per-lane counter copies (HH tables)

template <int DT>
struct QuadT;
template <>
struct QuadT<1> {
    int4 k;
    double2 a, b;
    __device__ __forceinline__ double v(int u) const { return u == 0 ? a.x : u == 1 ? a.y : u == 2 ? b.x : b.y; }
};
template <>
struct QuadT<0> {
    int4 k;
    float4 a;
    __device__ __forceinline__ float v(int u) const { return u == 0 ? a.x : u == 1 ? a.y : u == 2 ? a.z : a.w; }
};
__device__ __forceinline__ int kq(const int4 &k, int u) { return u == 0 ? k.x : u == 1 ? k.y : u == 2 ? k.z : k.w; }

// 4 rows from row r (VEC: 16-byte streaming loads; else scalar)
template <int DT, bool VEC>
__device__ __forceinline__ void load_quad(const int32_t *__restrict__ keys, const typename Fmt<DT>::V *__restrict__ vals,
                                          int64_t r, QuadT<DT> &q) {
    if (VEC) {
        q.k = __ldcs(reinterpret_cast<const int4 *>(keys + r));
        if constexpr (DT == 1) {
            q.a = __ldcs(reinterpret_cast<const double2 *>(vals + r));
            q.b = __ldcs(reinterpret_cast<const double2 *>(vals + r) + 1);
        } else {
            q.a = __ldcs(reinterpret_cast<const float4 *>(vals + r));
        }
    } else {
        q.k = make_int4(__ldcs(keys + r), __ldcs(keys + r + 1), __ldcs(keys + r + 2), __ldcs(keys + r + 3));
        if constexpr (DT == 1) {
            q.a = make_double2(__ldcs(vals + r), __ldcs(vals + r + 1));
            q.b = make_double2(__ldcs(vals + r + 2), __ldcs(vals + r + 3));
        } else {
            q.a = make_float4(__ldcs(vals + r), __ldcs(vals + r + 1), __ldcs(vals + r + 2), __ldcs(vals + r + 3));
        }
    }
}
// 4 rows from row r, vectorised when the row arrays are 16-byte aligned
template <int DT>
__device__ __forceinline__ void load_quad_rt(const int32_t *__restrict__ keys,
                                             const typename Fmt<DT>::V *__restrict__ vals, int64_t r, QuadT<DT> &q,
                                             bool vec) {
    if (vec) load_quad<DT, true>(keys, vals, r, q);
    else load_quad<DT, false>(keys, vals, r, q);
}
// up to 4 rows (fewer at the end of a range), scalar loads; missing rows are
// key 0, value 0
template <int DT>
__device__ __forceinline__ void load_partial(const int32_t *__restrict__ keys,
                                             const typename Fmt<DT>::V *__restrict__ vals, int64_t r, int cnt,
                                             QuadT<DT> &q) {
    using V = typename Fmt<DT>::V;
    int k[4] = {0, 0, 0, 0};
    V v[4] = {V(0), V(0), V(0), V(0)};
    for (int u = 0; u < cnt; ++u) { k[u] = keys[r + u]; v[u] = vals[r + u]; }
    q.k = make_int4(k[0], k[1], k[2], k[3]);
    if constexpr (DT == 1) { q.a = make_double2(v[0], v[1]); q.b = make_double2(v[2], v[3]); }
    else q.a = make_float4(v[0], v[1], v[2], v[3]);
}

// bulk prefetch of `bytes` (multiple of 16, 16-byte aligned) into L2
__device__ __forceinline__ void l2_prefetch(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint32_t atom_add_shared(uint32_t a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t atom_exch_shared(uint32_t a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

// Add a level sum T of group g at absolute level j into the slot table
// (slot j + K - 1; low 32 bits and high part in separate 64-bit words, so
// any number of partial sums adds without overflow).
template <int DT, int K>
__device__ __forceinline__ void slot_add(unsigned long long *slots, int64_t g, int j, int64_t T) {
    constexpr int NS = Fmt<DT>::KMAX + K;
    if (T == 0) return;
    unsigned long long *p = slots + ((size_t)g * NS + (j + K - 1)) * 2;
    atomicAdd(p, (unsigned long long)(T & 0xFFFFFFFFll));
    atomicAdd(p + 1, (unsigned long long)(T >> 32));
}

// value of counter word w (level w / LIMBS, limb w % LIMBS) as a level-sum part
template <int DT>
__device__ __forceinline__ int64_t counter_part(int w, uint32_t c) {
    if (Fmt<DT>::LIMBS == 2 && (w & 1)) return (int64_t)(int32_t)c * (int64_t)(1 << 20);
    return (int64_t)(int32_t)c;
}

// Shared memory of a table of G groups: counters u32 [CWB][gq], ktop int32
// [gr], knext int32 [gr], raised-group list int32 [gr]; gq = G + TAB_SINKS
// (one sink column per lane for the zero limbs of skipped rows) + the heavy
// groups' lane copies, rounded to 4; gr = G + 1 rounded to 4.  CWB = (K + XB) * LIMBS
// counter words per group: XB = 1 adds one level below the window for the
// band mode (Table::band_quad).
template <int DT, int K, int XB = 0>
struct TabGeom {
    static constexpr int LIMBS = Fmt<DT>::LIMBS;
    static constexpr int CW = K * LIMBS;
    static constexpr int CWB = (K + XB) * LIMBS;
    __host__ __device__ static int gq(int G, int nh = 0) { return (G + TAB_SINKS + 32 * nh + 3) & ~3; }
    __host__ __device__ static int gr(int G) { return (G + 1 + 3) & ~3; }
    __host__ __device__ static size_t bytes(int G, int nh = 0) {
        return (size_t)gq(G, nh) * 4 * CWB + (size_t)gr(G) * 12 + (nh ? (size_t)G + 4 * TAB_HMAX : 0);
    }
    // a table with the compile-time stride GQC >= gq(G): counters and the
    // per-group int arrays all GQC long
    __host__ __device__ static size_t bytes_gqc(int GQC) { return (size_t)GQC * (4 * CWB + 12); }
};

// One block's table.  Every method is entered by all threads of the block
// (slow_quad and finish contain barriers; fast_quad is barrier-free).
// GQC > 0: the counter-row stride is the compile-time constant GQC (>= gq(G)),
// so every atomic's counter offset is an immediate.
// HH: up to TAB_HMAX HEAVY groups (skewed keys, e.g. Zipf's head) get one
// counter copy per lane in streaming mode -- virtual group G + TAB_SINKS + 32 h +
// lane, always bank = lane -- because many lanes of a warp adding to one
// shared word serialise.  The copies are summed when published.
// XB = 1: BAND MODE for blocks whose groups do not share one window top
// (skewed keys leave most groups of a block untouched for a long time, values
// of several magnitudes give groups different tops).  After the first
// block-synchronous tile, such a block streams without barriers with all
// counters at window kuni = the largest top seen, spanning K + 1 levels
// kuni .. kuni - K: a row with k* = kuni or kuni - 1 deposits its K digits at
// its OWN window (shift s = kuni - k*: words (s + l) * LIMBS + h), which is
// exact through the absolute-level slot table whatever the group's final top
// (a row's digit at level j does not depend on the window, and a window at
// the row's own k* is never above the group's global top).  The group's top is
// tracked per row (shared atomicMax when it rises) for kglob.  Rows with k*
// outside the band go straight to the slot table (exceptional).  Once every
// group has reached kuni the block switches to the uniform mode (fast_quad),
// whose words are the same.
template <int DT, int K, int TPB, int GQC = 0, bool HH = false, int XB = 0>
struct Table {
    using F = Fmt<DT>;
    using V = typename F::V;
    using Geo = TabGeom<DT, K, XB>;
    static constexpr int CW = Geo::CW, LIMBS = Geo::LIMBS, CWB = Geo::CWB, NL = K + XB;
    static constexpr int ROWK = 32;          // s_mm words ROWK + k: rows of the first tile with k* = k
    static constexpr int NTOP = TAB_MM - 1;  // s_mm word: groups whose top reached kuni (band mode)
    static_assert(ROWK + F::KMAX < NTOP, "TAB_MM too small");

    uint32_t *cnt;
    int32_t *ktop, *knext;
    int *s_mm;  // TAB_MM shared words: [0], [1] raised-group list lengths (by call parity), [2 + k] groups at top k
    int32_t *rlist;  // raised groups of the current tile (shared, gq entries)
    int G, gq;
    int64_t gbase;  // global id of local group 0 (slot table / kglob index)
    int32_t *kglob;
    unsigned long long *slots;
    uint32_t cbase, wstride;
    int kuni;       // block-uniform window top (streaming mode) or -1
    uint32_t lim;   // magnitude bits limit of kuni's window
    uint32_t mlim;  // band mode: limit of window kuni - 1 (rows below it have k* < kuni)
    uint32_t llim;  // band mode: limit of window kuni - 2 (rows below it are outside the band)
    uint32_t big;   // OR of (old + 2^29) over observed counters
    bool first;
    bool band;      // band mode (XB = 1; block-uniform)
    int bcalls;     // band_quad calls since the last switch check (block-uniform)
    int bcheck;     // calls between switch checks (doubles after each failed check)
    int par;  // parity of slow_quad calls (block-uniform)
    int nh;           // heavy groups (HH)
    int8_t *hmap;     // local group -> heavy index or -1 (HH, shared, G entries)
    int32_t *hkey;    // heavy index -> local group (HH, shared, TAB_HMAX entries)
    Extractors<DT, K + XB> ex;

    __device__ __forceinline__ Table(unsigned char *mem, int *mm, int G_, int64_t gbase_, int32_t *kglob_,
                                     unsigned long long *slots_, int nh_ = 0)
        : s_mm(mm), G(G_), gbase(gbase_), kglob(kglob_), slots(slots_), kuni(-1), lim(0), mlim(0), llim(0), big(0),
          first(true), band(false), bcalls(0), bcheck(TAB_BAND_CHECK), par(0), nh(HH ? nh_ : 0), ex(0) {
        gq = GQC > 0 ? GQC : Geo::gq(G, nh);
        // (GQC > 0: the per-group int arrays are GQC long too -- compile-time
        // offsets; a G-dependent length costs the hot loop registers)
        const int gr = GQC > 0 ? GQC : Geo::gr(G);
        cnt = reinterpret_cast<uint32_t *>(mem);
        ktop = reinterpret_cast<int32_t *>(cnt + (size_t)CWB * gq);
        knext = ktop + gr;
        rlist = knext + gr;
        hkey = rlist + gr;
        hmap = reinterpret_cast<int8_t *>(hkey + TAB_HMAX);
        cbase = (uint32_t)__cvta_generic_to_shared(cnt);
        wstride = 4u * (uint32_t)gq;
    }
    // zero the table (caller: barrier before first use)
    __device__ __forceinline__ void clear() {
        for (int i = threadIdx.x; i < CWB * gq; i += TPB) cnt[i] = 0;
        for (int i = threadIdx.x; i < (GQC > 0 ? GQC : Geo::gr(G)); i += TPB) { ktop[i] = 0; knext[i] = 0; }
        for (int i = threadIdx.x; i < TAB_MM; i += TPB) s_mm[i] = i == 2 ? G : 0;  // all G groups at top 0
        if (HH && nh > 0)
            for (int i = threadIdx.x; i < G; i += TPB) hmap[i] = -1;
        kuni = -1;
        par = 0;
        lim = mlim = llim = 0;
        big = 0;
        first = true;
        band = false;
        bcalls = 0;
        bcheck = TAB_BAND_CHECK;
    }
    // set the heavy groups (HH; after clear() and a barrier, before a barrier)
    __device__ __forceinline__ void set_heavy(const int32_t *keys_local, int count) {
        if (!HH) return;
        for (int h = threadIdx.x; h < count && h < nh; h += TPB) {
            hkey[h] = keys_local[h];
            hmap[keys_local[h]] = (int8_t)h;
        }
    }
    // real group of a (virtual) group of the counter table
    __device__ __forceinline__ int real_group(int vg) const {
        return (HH && vg >= G + TAB_SINKS) ? hkey[(vg - G - TAB_SINKS) >> 5] : vg;
    }
    __device__ __forceinline__ void drain(int vg, int w, int kt) {
        const uint32_t c = atom_exch_shared(cbase + 4u * (uint32_t)vg + (uint32_t)w * wstride, 0u);
        if (c) slot_add<DT, K>(slots, gbase + real_group(vg), kt - w / LIMBS, counter_part<DT>(w, c));
    }
    // publish all counters of group g at window kt (no concurrent deposits);
    // the band level below the window is nonzero only in band mode, where
    // kt = kuni >= 1 (no level below -(K - 1) is ever deposited)
    __device__ __forceinline__ void publish_all(int g, int kt) {
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            int64_t T = 0;
#pragma unroll
            for (int h = 0; h < LIMBS; ++h) {
                const int w = l * LIMBS + h;
                uint32_t *p = cnt + (size_t)w * gq + g;
                T += counter_part<DT>(w, *p);
                *p = 0;
            }
            if (kt - l >= 1 - K) slot_add<DT, K>(slots, gbase + g, kt - l, T);
        }
    }

    // A row outside the streaming fast path: error bits, or (valid, k* above
    // kuni) deposited at its own window straight into the slot table.
    __device__ __forceinline__ void exceptional(int32_t k, V v, uint32_t &flags) {
        uint32_t f = 0;
        const int ks = kstar_of<DT>(v, f);
        if ((uint32_t)k >= (uint32_t)G) { flags |= FLAG_EKEY; return; }
        if (f) { flags |= f; return; }
        typename F::Digit d[K];
        digits_of<DT, K>(v, ks, d);
        atomicMax(&kglob[gbase + k], ks);
#pragma unroll
        for (int l = 0; l < K; ++l) slot_add<DT, K>(slots, gbase + k, ks - l, (int64_t)d[l]);
    }

    // Streaming deposit of 4 rows under kuni (kuni >= 0).  `in` bit u: row u
    // belongs to this table (others deposit zero limbs into the sink group).
    // Rows that fail the key / window check are handled one by one.
    // obs = false: the atomics return nothing (red.shared); legal on every
    // other call when TPB <= 256: once a counter passes 2^29 every thread adds
    // at most two more batches (an unobserved one and the observing one) before
    // it drains, so the counter stays below 2^29 + 2 * TPB * 4 * 2^19 < 2^31
    __device__ __forceinline__ void fast_quad(const QuadT<DT> &q, uint32_t in, uint32_t &flags, bool obs = true) {
        int32_t key[4];
        V val[4];
        uint32_t exc = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t k = kq(q.k, u);
            const V v = q.v(u);
            const uint32_t hw = DT == 1 ? (uint32_t)__double2hiint((double)v) << 1 : __float_as_uint((float)v) << 1;
            const bool iu = (in >> u) & 1u;
            const bool ok = iu && (uint32_t)k < (uint32_t)G && hw < lim;
            exc |= (iu && !ok) ? 1u << u : 0u;
            key[u] = ok ? k : G + (int)(threadIdx.x & 31);  // this lane's sink
            val[u] = ok ? v : V(0);
            if (HH && nh > 0 && ok) {  // a heavy group's row goes to this lane's copy
                const int hh = hmap[k];
                if (hh >= 0) key[u] = G + TAB_SINKS + 32 * hh + (int)(threadIdx.x & 31);
            }
        }
        uint32_t lo[4][K], hi[4][K], a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = cbase + 4u * (uint32_t)key[u];
            if (DT == 1) {
                double r = (double)val[u];
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    const double x = __hiloint2double(__double2hiint(r), __double2loint(r) | 1);  // reading A-1
                    const double t = __dadd_rn(x, (double)ex.e[l]);
                    const uint32_t tlo = (uint32_t)__double2loint(t);
                    const uint32_t thi = (uint32_t)__double2hiint(t);
                    lo[u][l] = (tlo & 0xFFFFFu) - 0x80000u;
                    hi[u][l] = __funnelshift_r(tlo, thi, 20) - ex.eb[l];
                    if (l + 1 < K) r = __dsub_rn(r, __dsub_rn(t, (double)ex.e[l]));
                }
            } else {
                float r = (float)val[u];
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    const float x = __uint_as_float(__float_as_uint(r) | 1u);
                    const float t = __fadd_rn(x, (float)ex.e[l]);
                    lo[u][l] = __float_as_uint(t) - ex.eb[l];
                    hi[u][l] = 0;
                    if (l + 1 < K) r = __fsub_rn(r, __fsub_rn(t, (float)ex.e[l]));
                }
            }
        }
        // one atomic per counter position and row; positions the whole warp
        // leaves at zero are skipped (one vote)
#pragma unroll
        for (int l = 0; l < K; ++l) {
#pragma unroll
            for (int h = 0; h < LIMBS; ++h) {
                uint32_t any = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) any |= h ? hi[u][l] : lo[u][l];
                // (low limbs of a batch are almost never all zero: no vote unless TAB_VOTE_LO)
                if ((LIMBS == 2 && h == 0 && !TAB_VOTE_LO) || __any_sync(0xffffffffu, any != 0u)) {
                    const uint32_t off = (uint32_t)(LIMBS * l + h) * (GQC > 0 ? 4u * GQC : wstride);
                    if (TPB <= 256 && !obs) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) red_shared(a[u] + off, h ? hi[u][l] : lo[u][l]);
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            big |= atom_add_shared(a[u] + off, h ? hi[u][l] : lo[u][l]) + TAB_DRAIN_BIAS;
                    }
                }
            }
        }
        if (big & TAB_DRAIN_MASK) {  // rare: drain every counter of this batch that is past 2^29
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if ((uint32_t)(key[u] - G) < (uint32_t)TAB_SINKS) continue;  // a sink
#pragma unroll
                for (int w = 0; w < CW; ++w) {
                    const uint32_t c = ld_shared_u32(a[u] + (uint32_t)w * wstride);
                    if ((c + TAB_DRAIN_BIAS) & TAB_DRAIN_MASK) drain(key[u], w, kuni);
                }
            }
            big = 0;
        }
        while (exc) {
            const int u = __ffs(exc) - 1;
            exc &= exc - 1;
            exceptional(kq(q.k, u), q.v(u), flags);
        }
    }

    // Band-mode deposit of 4 rows (XB = 1, kuni >= 1): a row with k* = kuni
    // - s, s in {0, 1}, deposits its digits at its own window into counter
    // words (s + l) * LIMBS + h; its group's tracked top rises to k* (shared
    // atomicMax, only when it rises; NTOP counts the groups at kuni).  Rows
    // outside the band, bad keys and non-finite values are handled one by one.
    __device__ __forceinline__ void band_quad(const QuadT<DT> &q, uint32_t in, uint32_t &flags) {
        int32_t key[4];
        V val[4];
        uint32_t sh[4];
        uint32_t exc = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t k = kq(q.k, u);
            const V v = q.v(u);
            const uint32_t hw = DT == 1 ? (uint32_t)__double2hiint((double)v) << 1 : __float_as_uint((float)v) << 1;
            const bool iu = (in >> u) & 1u;
            const bool ok = iu && (uint32_t)k < (uint32_t)G && hw < lim && hw >= llim;
            exc |= (iu && !ok) ? 1u << u : 0u;
            const uint32_t s_ = hw < mlim ? 1u : 0u;
            key[u] = ok ? k : G + (int)(threadIdx.x & 31);  // this lane's sink
            val[u] = ok ? v : V(0);
            sh[u] = ok ? s_ : 0u;
            if (ok) {
                const int kr = kuni - (int)s_;
                if (kr > ktop[k]) {
                    const int old = atomicMax(&ktop[k], kr);
                    if (old < kuni && kr == kuni) atomicAdd(&s_mm[NTOP], 1);
                }
                if (HH && nh > 0) {
                    const int hh = hmap[k];
                    if (hh >= 0) key[u] = G + TAB_SINKS + 32 * hh + (int)(threadIdx.x & 31);
                }
            }
        }
        const uint32_t ws = GQC > 0 ? 4u * GQC : wstride;
        uint32_t lo[4][K], hi[4][K], a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = cbase + 4u * (uint32_t)key[u] + sh[u] * (uint32_t)LIMBS * ws;
            const bool s1 = sh[u] != 0u;
            if (DT == 1) {
                double r = (double)val[u];
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    const double e = s1 ? (double)ex.e[l + XB] : (double)ex.e[l];
                    const uint32_t eb = s1 ? ex.eb[l + XB] : ex.eb[l];
                    const double x = __hiloint2double(__double2hiint(r), __double2loint(r) | 1);  // reading A-1
                    const double t = __dadd_rn(x, e);
                    const uint32_t tlo = (uint32_t)__double2loint(t);
                    const uint32_t thi = (uint32_t)__double2hiint(t);
                    lo[u][l] = (tlo & 0xFFFFFu) - 0x80000u;
                    hi[u][l] = __funnelshift_r(tlo, thi, 20) - eb;
                    if (l + 1 < K) r = __dsub_rn(r, __dsub_rn(t, e));
                }
            } else {
                float r = (float)val[u];
#pragma unroll
                for (int l = 0; l < K; ++l) {
                    const float e = s1 ? (float)ex.e[l + XB] : (float)ex.e[l];
                    const uint32_t eb = s1 ? ex.eb[l + XB] : ex.eb[l];
                    const float x = __uint_as_float(__float_as_uint(r) | 1u);
                    const float t = __fadd_rn(x, e);
                    lo[u][l] = __float_as_uint(t) - eb;
                    hi[u][l] = 0;
                    if (l + 1 < K) r = __fsub_rn(r, __fsub_rn(t, e));
                }
            }
        }
#pragma unroll
        for (int l = 0; l < K; ++l) {
#pragma unroll
            for (int h = 0; h < LIMBS; ++h) {
                uint32_t any = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) any |= h ? hi[u][l] : lo[u][l];
                if ((LIMBS == 2 && h == 0 && !TAB_VOTE_LO) || __any_sync(0xffffffffu, any != 0u)) {
                    const uint32_t off = (uint32_t)(LIMBS * l + h) * ws;
#pragma unroll
                    for (int u = 0; u < 4; ++u) big |= atom_add_shared(a[u] + off, h ? hi[u][l] : lo[u][l]) + TAB_DRAIN_BIAS;
                }
            }
        }
        if (big & TAB_DRAIN_MASK) {  // rare: drain every counter of this batch's groups that is past 2^29
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if ((uint32_t)(key[u] - G) < (uint32_t)TAB_SINKS) continue;  // a sink
                const uint32_t g0 = cbase + 4u * (uint32_t)key[u];
#pragma unroll
                for (int w = 0; w < CWB; ++w) {
                    const uint32_t c = ld_shared_u32(g0 + (uint32_t)w * wstride);
                    if ((c + TAB_DRAIN_BIAS) & TAB_DRAIN_MASK) drain(key[u], w, kuni);
                }
            }
            big = 0;
        }
        while (exc) {
            const int u = __ffs(exc) - 1;
            exc &= exc - 1;
            exceptional(kq(q.k, u), q.v(u), flags);
        }
        // once every group has reached kuni, the uniform mode takes over
        // (same counter words; block-uniform decision).  Checked after
        // TAB_BAND_CHECK calls, then at doubling intervals: with skewed keys
        // some groups may never reach the top, and each check is a barrier
        if (++bcalls == bcheck) {
            bcalls = 0;
            if (__syncthreads_and(ld_shared_u32((uint32_t)__cvta_generic_to_shared(&s_mm[NTOP])) >= (uint32_t)G))
                band = false;
            else
                bcheck = min(2 * bcheck, TAB_BAND_CHECK_MAX);
        }
    }

    // set the window limits for top kuni (block-uniform)
    __device__ __forceinline__ void set_window(int ku) {
        kuni = ku;
        ex = Extractors<DT, K + XB>(kuni);
        auto limit = [](int k) {
            return (uint32_t)(F::W * k + F::W - 1 - F::m + F::BIAS) << (F::m % 32 + 1);
        };
        lim = limit(kuni);
        mlim = kuni >= 1 ? limit(kuni - 1) : 0u;
        llim = kuni >= 2 ? limit(kuni - 2) : 0u;
    }

    // Block-synchronous deposit of 4 rows (row u taken when bit u of `in`):
    // per-row k*, raise the groups' tops, publish a raised group's counters at
    // its old window, then deposit each row at its group's window.  May switch
    // the table to streaming mode (kuni >= 0, block-uniform).
    __device__ __forceinline__ void slow_quad(const QuadT<DT> &q, uint32_t in, uint32_t &flags) {
        const int tid = threadIdx.x;
        int32_t key[4];
        int changed = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int ks;
            key[u] = check_row<DT>(kq(q.k, u), q.v(u), (in >> u) & 1u, G, flags, ks);
            if (XB > 0 && first && key[u] >= 0) atomicAdd(&s_mm[ROWK + ks], 1);
            if (key[u] >= 0 && ks > ktop[key[u]]) {
                // the thread whose atomicMax first lifts knext above ktop lists the group
                const int old = atomicMax(&knext[key[u]], ks);
                if (old == ktop[key[u]]) rlist[atomicAdd(&s_mm[par], 1)] = key[u];
                changed = 1;
            }
        }
        const int any = __syncthreads_or(changed) | (first ? 1 : 0);
        first = false;
        // the other parity's list length was last read before the previous
        // call's second barrier and is next appended to after this call's
        if (tid == 0) s_mm[par ^ 1] = 0;
        if (any) {
            // raised groups only: publish at the old window, move the top, and
            // keep the number of groups per window top (s_mm[1 + k])
            const int nr = s_mm[par];
            for (int i = tid; i < nr; i += TPB) {
                const int g = rlist[i];
                publish_all(g, ktop[g]);
                atomicSub(&s_mm[2 + ktop[g]], 1);
                atomicAdd(&s_mm[2 + knext[g]], 1);
                ktop[g] = knext[g];
            }
            __syncthreads();
            int ku = -1, kb = 1, best = -1;
            for (int k = 0; k <= F::KMAX; ++k) {
                if (s_mm[2 + k] == G) ku = k;
                // band top: the pair of window tops {k - 1, k} covering the
                // most rows of the first tile; on a tie the pair whose top
                // holds more rows (a top no row reached would keep every
                // group below it, in band mode for good)
                const int pr = s_mm[ROWK + k] + (k >= 1 ? s_mm[ROWK + k - 1] : 0);
                if (k >= 1 && (pr > best || (pr == best && s_mm[ROWK + k] > s_mm[ROWK + kb]))) { best = pr; kb = k; }
            }
            if (ku >= 0) {
                set_window(ku);
            } else if (XB > 0) {
                // groups at different tops: band mode.  Every group's
                // counters go out at its own window first; the rows of this
                // call go straight to the slot table below.
                for (int g = tid; g < G; g += TPB) publish_all(g, ktop[g]);
                if (tid == 0) {
                    int at = 0;  // groups whose top is already >= kb
                    for (int k = kb; k <= F::KMAX; ++k) at += s_mm[2 + k];
                    s_mm[NTOP] = at;
                }
                set_window(kb);
                band = true;
                bcalls = 0;
                bcheck = TAB_BAND_CHECK;
            }
        }
        __syncthreads();  // raise phase done / the list length is reset before the next call's appends
        par ^= 1;
        if (XB > 0 && band) {  // this call's rows, at their groups' windows (>= their k*)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (key[u] < 0) continue;
                const int kt = ktop[key[u]];
                typename F::Digit d[K];
                digits_of<DT, K>(q.v(u), kt, d);
#pragma unroll
                for (int l = 0; l < K; ++l) slot_add<DT, K>(slots, gbase + key[u], kt - l, (int64_t)d[l]);
            }
            return;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (key[u] < 0) continue;
            const int kt = ktop[key[u]];
            uint32_t lo[K], hi[K];
            row_limbs<DT, K>(F::mul(q.v(u), F::pow2(F::m - F::W * kt)), lo, hi);
            const uint32_t a = cbase + 4u * (uint32_t)key[u];
#pragma unroll
            for (int l = 0; l < K; ++l)
#pragma unroll
                for (int h = 0; h < LIMBS; ++h) {
                    const uint32_t old = atom_add_shared(a + (uint32_t)(LIMBS * l + h) * wstride, h ? hi[l] : lo[l]);
                    if ((old + TAB_DRAIN_BIAS) & TAB_DRAIN_MASK) drain(key[u], LIMBS * l + h, kt);
                }
        }
    }

    // block-uniform: the table streams in the uniform mode (fast_quad) from
    // now on (callers may then call fast_quad directly in a loop of its own)
    __device__ __forceinline__ bool uniform() const { return kuni >= 0 && !(XB > 0 && band); }

    __device__ __forceinline__ void quad(const QuadT<DT> &q, uint32_t in, uint32_t &flags, bool obs = true) {
#if TAB_DEBUG
        ++dbg[(XB > 0 && band) ? 1 : kuni >= 0 ? 2 : 0];
#endif
        if (XB > 0 && band) band_quad(q, in, flags);
        else if (kuni >= 0) fast_quad(q, in, flags, obs);
        else slow_quad(q, in, flags);
    }
#if TAB_DEBUG
    unsigned dbg[3] = {0, 0, 0};  // calls in slow / band / uniform mode (this thread)
    __device__ __forceinline__ void dbg_flush(unsigned long long *out) {
        if (threadIdx.x == 0)
            for (int i = 0; i < 3; ++i) atomicAdd(out + i, (unsigned long long)dbg[i]);
    }
#endif

    // publish every group's counters at its block window and raise the
    // global tops; leaves the table zeroed (barriers on both sides)
    __device__ __forceinline__ void finish() {
        __syncthreads();
        for (int g = threadIdx.x; g < G; g += TPB) {
            // streaming modes: every counter is at window kuni (band mode:
            // ktop is the tracked top); block-synchronous: at ktop
            publish_all(g, kuni >= 0 ? kuni : ktop[g]);
            if (ktop[g] > 0) atomicMax(&kglob[gbase + g], ktop[g]);
        }
        if (HH && nh > 0 && kuni >= 0) {  // the lane copies hold digits under kuni
            for (int i = threadIdx.x; i < nh * CWB; i += TPB) {
                const int h = i / CWB, w = i - h * CWB;
                int64_t T = 0;
                uint32_t *p = cnt + (size_t)w * gq + G + TAB_SINKS + 32 * h;
                for (int l = 0; l < 32; ++l) {
                    T += counter_part<DT>(w, p[l]);
                    p[l] = 0;
                }
                slot_add<DT, K>(slots, gbase + hkey[h], kuni - w / LIMBS, T);
            }
        }
        __syncthreads();
    }
};

}  // namespace repro
