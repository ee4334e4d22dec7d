// k_route.cu -- the GroupBy for group counts above one SM's table (SURVEY.md
// section 8 rows a4/a5), in ONE pass over the rows' bytes.
//
// PartitionAndAggregate (Alg. 4) splits the groups into
// partitions whose tables fit the fast memory (F = f^d)
// and moves every row to its partition before aggregating.  The two-pass sweep
// (k_sweep.cu) moves rows through HBM (12 B read + 12 B written + 12 B read
// again per binary64 row on top of the input).  Here the moving is done
// through L2 instead, with every SM both a PRODUCER and a CONSUMER at once:
//   * the groups are split into Q partitions by g mod Q (the local id is
//     g / Q; `mod` spreads the hot keys of skewed data); partition q lives in
//     the shared-memory table of R = floor(SMs / Q) consumer blocks
//     q + Q r, and producer block b sends its partition-q rows to consumer
//     q + Q (b mod R);
//   * producer warps stream their block's contiguous row range from HBM
//     once, rank each tile's rows by partition (warp match + shared
//     atomics), stage them in partition order and append each partition's
//     run to its consumer's RING (a small global buffer that stays in L2:
//     8192 rows per consumer);
//   * consumer warps read their ring in order and deposit the rows into the
//     block's table (32-bit limb counters, table_core.cuh arithmetic);
//   * the few HEAVY keys of skewed data (sampled, >= 1/512 of the rows each)
//     are never routed: producers deposit them into per-lane counter copies
//     of their own block (one SM would otherwise receive, e.g., 12% of all
//     rows for Zipf's top key).
// Both tables publish into the ABSOLUTE-LEVEL slot table (kglob, slots) that
// k_fold (k_state.cu) turns into canonical states and Eq. 1 read-outs, so the
// bits do not depend on which block deposited which row.
//
// Window tops (Alg. 1 lines 3-9) without any block-level
// bookkeeping: a sampled BAND of window tops {kb - XB .. kb} (XB = 0 or 1) is
// chosen once; a row whose k* = kb - s lies in the band deposits its K digits
// at its OWN window into counter words (s + l) * LIMBS + h, which is exact
// through the absolute-level slot table (a row's digit at level j does not
// depend on the window, and a window at the row's own k* never lies above
// its group's final top).  Two bits per group record which tops its rows
// reached (-> kglob).  Rows outside the band (rare by construction) are
// deposited one by one straight into the slot table.
//
// Ring protocol (per consumer c; positions are 64-bit and only grow):
//   * a producer reserves a run [pos, pos + cnt) with one atomicAdd on
//     tail[c], and writes it once head[c] >= pos + cnt - RING (every row of
//     the previous lap in those slots has been consumed): values first, a
//     fence, then the keys carrying the lap's parity in bit 31 -- a key with
//     the expected parity below the current tail is a written row;
//   * a producer never waits on one consumer while it holds rows for another
//     that it could write: each pass over a staged tile writes every run
//     whose ring has room, so a consumer is only ever waiting for rows whose
//     writer is waiting for that same consumer -- which frees the room;
//   * consumer warps take batches of 128 positions round-robin, at most
//     RING / 256 batches ahead of the slowest one (so a slot seen with the
//     expected parity cannot be two laps old), and publish head = the first
//     unconsumed position (atomicMax) as they go;
//   * the end: producers finished (done == blocks, after a fence) makes tail
//     final; positions at or past it never come.
// STATUS: opt-in (repro_set_route_mode(1)).  Bit-exact against the oracle
// (tests/test_gpu_route.py), and the rings never reach HBM (ncu: 4 MB of DRAM
// writes for 2^26 binary64 rows), but measured SLOWER than the two-pass sweep
// on B200 (2^28 rows, 65536 groups: 5.3 ms vs 3.1 ms): the producer loop is
// latency-bound (per-tile barriers with only 24 KB of row loads in flight per
// SM: 2.1 ms even without any ring traffic), and the ring handshakes add more.
//
// Every wait polls with a bound; a wait that exceeds it sets FLAG_ESTALL
// (REPRO_ECUDA) and every block leaves instead of hanging the GPU.  All
// blocks must be resident at once: the kernel is launched cooperatively with
// one block per SM.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"
#include "table_core.cuh"

#include <algorithm>

namespace repro {

namespace {

#ifndef RT_RING_LOG
#define RT_RING_LOG 14  // rows per consumer ring: 16384 (148 rings of binary64 rows: 39 MB of L2)
#endif
#ifndef RT_L2PF
#define RT_L2PF 0  // 1: lane 0 of each producer warp bulk-prefetches its rows two tiles ahead into L2
#endif
#ifndef RT_LATE_LOAD
#define RT_LATE_LOAD 0  // 1: the next tile's row loads are issued after the reservation atomics
#endif
#ifndef RT_DIAG
#define RT_DIAG 0  // diagnostics only (wrong sums): 1 producers skip reservations and ring writes
#endif
#ifndef RT_PWARPS
#define RT_PWARPS 8     // producer warps (the rest of the block consumes)
#endif
constexpr int RT_TPB = 512;
constexpr int RT_PW = RT_PWARPS;
constexpr int RT_CWN = RT_TPB / 32 - RT_PW;  // consumer warps
constexpr int RT_PT = RT_PW * 32;            // producer threads
constexpr int RT_QPT = 2;                    // quads per producer thread per tile
constexpr int RT_TILE = 4 * RT_QPT * RT_PT;  // rows per producer tile
constexpr int RT_RING = 1 << RT_RING_LOG;
constexpr int RT_BATCH = 128;                // consumer batch: one quad per lane
constexpr int RT_LEAD = RT_RING / RT_BATCH / 2;
constexpr int RT_PUB = 1024;                 // head publication step (rows)
constexpr int RT_QMAX = 160;                 // partitions (>= the SM count; one producer thread each)
constexpr int RT_NH = 32;                    // heavy keys
constexpr int RT_HCOLS = RT_NH * 32 + 32;    // heavy lane copies + per-lane sinks
constexpr int RT_HSLOTS = 64;                // heavy-key hash
constexpr int RT_SAMPLE = 8192;
constexpr int RT_SHASH = 16384;              // sample counting hash (int2 slots)
constexpr long long RT_SPIN = 1ll << 22;     // polls (>= 64 ns each) before a wait gives up
#ifndef RT_PROF
#define RT_PROF 0  // debug builds: cycles per phase (repro_debug_route_prof)
#endif
#if RT_PROF
__device__ unsigned long long g_rt_prof[16];
#define RT_T0() long long rt_t0_ = clock64()
#define RT_T(i) do { const long long t_ = clock64(); rt_acc[i] += t_ - rt_t0_; rt_t0_ = t_; } while (0)
#define RT_C(i) (++rt_acc[i])
#else
#define RT_T0() do {} while (0)
#define RT_T(i) do {} while (0)
#define RT_C(i) do {} while (0)
#endif
enum { RC_KB = 0, RC_NH = 1, RC_DONE = 2, RC_ABORT = 3, RC_HKEY = 8, RC_WORDS = 8 + RT_NH };
static_assert(RT_QMAX <= RT_PT, "one producer thread per partition");
static_assert(RT_RING >= 2 * RT_TILE + RT_PUB + RT_BATCH * RT_LEAD / 2, "ring too small for the wait bounds");

template <int DT, int K, int XB>
struct RtGeo {
    using V = typename Fmt<DT>::V;
    static constexpr int LIMBS = Fmt<DT>::LIMBS, CWB = (K + XB) * LIMBS;
    static constexpr size_t fixed() {
        return (size_t)RT_QMAX * (8 + 8 + 8 + 4 + 4 + 4 + 4)  // run positions, cached heads, reservation ends, counts, lengths, states, positions
               + (size_t)RT_HSLOTS * 8 + RT_NH * 4          // heavy hash, heavy tops
               + (size_t)CWB * RT_HCOLS * 4 + 64;           // heavy lane copies
    }
    // counter columns gq (local groups + sink, multiple of 4)
    static constexpr size_t bytes(int gq) { return fixed() + (size_t)CWB * gq * 4 + (size_t)((gq + 15) / 16) * 4; }
};

template <int DT>
struct RtArgs {
    const int32_t *keys;
    const typename Fmt<DT>::V *vals;
    int64_t n;
    int32_t G;
    int Q, R, S;                // partitions, consumers per partition, blocks
    uint32_t M;                 // g / Q = umulhi(g, M) for g < G (M = ceil(2^32 / Q), G Q < 2^32)
    int gq;                     // counter columns of a table
    unsigned long long *ring;   // rings [S][RING][RT_W<DT>] (tagged words)
    unsigned long long *tail, *head;  // [S * RT_PADW] (one 128-byte line each)
    int32_t *ctrl, *kglob;
    unsigned long long *slots;
    uint32_t *status;
};

// Ring slots hold 64-bit words whose bit 63 is the lap parity of the
// position (1 on lap 0: the ring starts zeroed).  binary64 row: w0 = tag |
// local key << 32 | low value word, w1 = tag | high value word; binary32 row:
// w0 = tag | local key << 32 | value bits.  Aligned 64-bit accesses are
// single-copy atomic, so a row whose words all carry the expected tag is the
// row of this lap, whole -- no fence between writer and reader.
template <int DT>
constexpr int RT_W = DT == 1 ? 2 : 1;
constexpr int RT_PADW = 16;  // tail / head stride (words)
__device__ __forceinline__ unsigned long long lap_tag(unsigned long long p) {
    return ((~(p >> RT_RING_LOG)) & 1ull) << 63;
}
__device__ __forceinline__ void st_v2_u64(unsigned long long *p, unsigned long long a, unsigned long long b) {
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" :: "l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_u64(unsigned long long *p, unsigned long long a) {
    asm volatile("st.global.u64 [%0], %1;" :: "l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ void ld_vol_v2_u64(const unsigned long long *p, unsigned long long &a,
                                              unsigned long long &b) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long ld_vol_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_vol_i32(const int32_t *p) {
    int v;
    asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void atom_or_shared(uint32_t a, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" :: "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void pbar() { asm volatile("bar.sync 1, %0;" :: "n"(RT_PT) : "memory"); }
// producer-group barrier returning how many producer threads passed p
__device__ __forceinline__ int pbar_count(bool p) {
    int r;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tbarrier.red.popc.u32 %0, 1, %2, q;\n\t}"
                 : "=r"(r) : "r"((int)p), "n"(RT_PT) : "memory");
    return r;
}
__device__ __forceinline__ int heavy_of(const int2 *hh, int32_t k) {
    uint32_t h = ((uint32_t)k * 0x9E3779B1u) >> 26;
    for (;;) {
        const int2 e = hh[h];
        if (e.x == k) return e.y;
        if (e.x == -1) return -1;
        h = (h + 1) & (RT_HSLOTS - 1);
    }
}

// 1. sample: heavy keys (>= 1/512 of RT_SAMPLE evenly spaced rows, at most
// RT_NH) and the band top kb (the top, or pair of tops with XB, holding the
// most sampled rows).  Performance only: any choice gives the same bits.
template <int DT>
__global__ void __launch_bounds__(1024) k_rt_sample(const int32_t *__restrict__ keys,
                                                    const typename Fmt<DT>::V *__restrict__ vals, int64_t n,
                                                    int32_t G, int xb, int32_t *ctrl) {
    extern __shared__ int2 hs[];  // (key, count), key -1 = empty
    __shared__ int kc[32];
    __shared__ int s_nh;
    const int tid = threadIdx.x;
    for (int i = tid; i < RT_SHASH; i += 1024) hs[i] = make_int2(-1, 0);
    if (tid < 32) kc[tid] = 0;
    if (tid == 0) s_nh = 0;
    __syncthreads();
    for (int i = tid; i < RT_SAMPLE; i += 1024) {
        const int64_t r = n * i / RT_SAMPLE;
        if (r >= n) continue;
        const int32_t k = keys[r];
        if ((uint32_t)k >= (uint32_t)G) continue;
        uint32_t f = 0;
        const int ks = kstar_of<DT>(vals[r], f);
        if (ks >= 0) atomicAdd(&kc[ks], 1);
        uint32_t h = ((uint32_t)k * 0x9E3779B1u) >> (32 - 14);
        for (;;) {
            const int old = atomicCAS(&hs[h].x, -1, k);
            if (old == -1 || old == k) { atomicAdd(&hs[h].y, 1); break; }
            h = (h + 1) & (RT_SHASH - 1);
        }
    }
    __syncthreads();
    const int samples = (int)min((int64_t)RT_SAMPLE, n);
    const int thr = max(4, samples / 512);
    for (int i = tid; i < RT_SHASH; i += 1024)
        if (hs[i].x >= 0 && hs[i].y >= thr) {
            const int s = atomicAdd(&s_nh, 1);
            if (s < RT_NH) ctrl[RC_HKEY + s] = hs[i].x;
        }
    __syncthreads();
    if (tid == 0) {
        ctrl[RC_NH] = min(s_nh, RT_NH);
        int kb = 0, best = -1;
        for (int k = 0; k <= Fmt<DT>::KMAX; ++k) {
            const int sc = kc[k] + ((xb && k >= 1) ? kc[k - 1] : 0);
            if (sc > best) { best = sc; kb = k; }
        }
        ctrl[RC_KB] = kb;
    }
}

// 2. the routed pass (one block per SM, cooperative launch)
template <int DT, int K, int XB>
__global__ void __launch_bounds__(RT_TPB, 1) k_route(RtArgs<DT> A) {
    using F = Fmt<DT>;
    using V = typename F::V;
    using Geo = RtGeo<DT, K, XB>;
    constexpr int LIMBS = F::LIMBS, CWB = Geo::CWB, NL = K + XB;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_cprog[RT_CWN];
    __shared__ unsigned long long s_pub;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    const int Q = A.Q, gq = A.gq;
#if RT_PROF
    long long rt_acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif

    // shared memory carve
    unsigned long long *qpos = reinterpret_cast<unsigned long long *>(smem);
    unsigned long long *hcache = qpos + RT_QMAX;
    int2 *hhash = reinterpret_cast<int2 *>(hcache + 2 * RT_QMAX);
    int32_t *qcnt = reinterpret_cast<int32_t *>(hhash + RT_HSLOTS);
    int32_t *qoff = qcnt + RT_QMAX;
    int32_t *qst = qoff + RT_QMAX;  // run state per partition: 1 = written this tile
    uint32_t *qpos32 = reinterpret_cast<uint32_t *>(qst + RT_QMAX);  // low words of qpos
    unsigned long long *lend = hcache + RT_QMAX;  // end of each partition's last reservation
    uint32_t *htop = qpos32 + RT_QMAX;
    uint32_t *hcnt = htop + RT_NH;                      // [CWB][RT_HCOLS]
    uint32_t *cnt = hcnt + (size_t)CWB * RT_HCOLS;      // [CWB][gq]
    uint32_t *topb = cnt + (size_t)CWB * gq;            // 2 bits per local group

    const int kb = A.ctrl[RC_KB];
    const int nh = A.ctrl[RC_NH];
    for (int i = tid; i < CWB * gq; i += RT_TPB) cnt[i] = 0;
    for (int i = tid; i < (gq + 15) / 16; i += RT_TPB) topb[i] = 0;
    for (int i = tid; i < CWB * RT_HCOLS; i += RT_TPB) hcnt[i] = 0;
    for (int i = tid; i < RT_NH; i += RT_TPB) htop[i] = 0;
    for (int i = tid; i < RT_HSLOTS; i += RT_TPB) hhash[i] = make_int2(-1, -1);
    for (int i = tid; i < RT_QMAX; i += RT_TPB) { qcnt[i] = 0; hcache[i] = 0; lend[i] = 0; qst[i] = 0; }
    if (tid < RT_CWN) s_cprog[tid] = tid;
    if (tid == 0) s_pub = 0;
    __syncthreads();
    if (tid == 0)
        for (int h = 0; h < nh; ++h) {
            const int32_t k = A.ctrl[RC_HKEY + h];
            uint32_t s = ((uint32_t)k * 0x9E3779B1u) >> 26;
            while (hhash[s].x != -1) s = (s + 1) & (RT_HSLOTS - 1);
            hhash[s] = make_int2(k, h);
        }
    __syncthreads();

    // the band: rows with llim <= |b| bits < lim have k* in {kb - XB .. kb};
    // shift s = 1 when below mlim (k* = kb - 1)
    auto limit = [](int k) { return (uint32_t)(F::W * k + F::W - 1 - F::m + F::BIAS) << (F::m % 32 + 1); };
    const uint32_t lim = limit(kb);
    const uint32_t mlim = kb >= 1 ? limit(kb - 1) : 0u;
    const uint32_t llim = XB ? (kb >= 2 ? limit(kb - 2) : 0u) : mlim;
    const Extractors<DT, NL> ex(kb);
    uint32_t flags = 0;
    uint32_t big = 0;

    // this block as a consumer: partition qown, global id of local group j = j Q + qown
    const bool cons = b < Q * A.R;
    const int qown = cons ? b % Q : 0;
    const int gb = cons ? (A.G - qown + Q - 1) / Q : 0;  // local groups

    // a row outside the band: error bits, or its digits at its own window
    // straight into the slot table
    auto exceptional = [&](int64_t g, V v) {
        uint32_t f = 0;
        const int ks = kstar_of<DT>(v, f);
        if (f) { flags |= f; return; }
        typename F::Digit d[K];
        digits_of<DT, K>(v, ks, d);
        atomicMax(&A.kglob[g], ks);
#pragma unroll
        for (int l = 0; l < K; ++l) slot_add<DT, K>(A.slots, g, ks - l, (int64_t)d[l]);
    };
    // Deposit the rows u of a quad with bit u of `in` into the table at
    // shared address tbase (column stride 4 B, word stride ws), column
    // col[u]; sink[u] takes a row that is not deposited.  gid(col) is the
    // group of a column; mark(col, bit) records the row's top.
    auto deposit = [&](uint32_t tbase, uint32_t ws, const int (&colin)[4], const int (&sink)[4], const V (&v)[4],
                       uint32_t in, auto &&gid, auto &&mark) {
        int col[4];
        V val[4];
        uint32_t sh[4];
        uint32_t exc = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t hw = DT == 1 ? (uint32_t)__double2hiint((double)v[u]) << 1 : __float_as_uint((float)v[u]) << 1;
            const bool iu = (in >> u) & 1u;
            const bool ok = iu && hw < lim && hw >= llim;
            const uint32_t s_ = (XB && hw < mlim) ? 1u : 0u;
            exc |= (iu && !ok) ? 1u << u : 0u;
            col[u] = ok ? colin[u] : sink[u];
            val[u] = ok ? v[u] : V(0);
            sh[u] = ok ? s_ : 0u;
            if (ok) mark(colin[u], s_ ? 1u : 2u);
        }
        uint32_t lo[4][K], hi[4][K], a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = tbase + 4u * (uint32_t)col[u] + sh[u] * (uint32_t)LIMBS * ws;
            const bool s1 = XB && sh[u] != 0u;
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
                if (__any_sync(0xffffffffu, any != 0u)) {
                    const uint32_t off = (uint32_t)(LIMBS * l + h) * ws;
#pragma unroll
                    for (int u = 0; u < 4; ++u) big |= atom_add_shared(a[u] + off, h ? hi[u][l] : lo[u][l]) + TAB_DRAIN_BIAS;
                }
            }
        }
        if (big & TAB_DRAIN_MASK) {  // rare: drain every counter of this quad's columns past 2^29
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (col[u] == sink[u]) continue;
                const uint32_t c0 = tbase + 4u * (uint32_t)col[u];
#pragma unroll
                for (int w = 0; w < CWB; ++w) {
                    const uint32_t c = ld_shared_u32(c0 + (uint32_t)w * ws);
                    if ((c + TAB_DRAIN_BIAS) & TAB_DRAIN_MASK) {
                        const uint32_t t = atom_exch_shared(c0 + (uint32_t)w * ws, 0u);
                        if (t) slot_add<DT, K>(A.slots, gid(col[u]), kb - w / LIMBS, counter_part<DT>(w, t));
                    }
                }
            }
            big = 0;
        }
        if (exc) {  // rare (constant indices: the row arrays stay in registers)
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if ((exc >> u) & 1u) exceptional(gid(colin[u]), v[u]);
        }
    };
    const uint32_t cbase = (uint32_t)__cvta_generic_to_shared(cnt);
    const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(hcnt);
    const uint32_t cws = 4u * (uint32_t)gq, hws = 4u * (uint32_t)RT_HCOLS;
    auto gid_local = [&](int col) { return (int64_t)col * Q + qown; };
    auto gid_heavy = [&](int col) { return (int64_t)A.ctrl[RC_HKEY + (col >> 5)]; };
    auto mark_local = [&](int col, uint32_t bit) {
        const uint32_t sb = bit << ((col & 15) * 2);
        if (!(topb[col >> 4] & sb)) atom_or_shared((uint32_t)__cvta_generic_to_shared(&topb[col >> 4]), sb);
    };
    auto mark_heavy = [&](int col, uint32_t bit) {
        if (!(htop[col >> 5] & bit)) atom_or_shared((uint32_t)__cvta_generic_to_shared(&htop[col >> 5]), bit);
    };

    if (warp < RT_PW) {
        // ---------------- producer ----------------
        const int ptid = tid;
        int64_t chunk = (A.n + A.S - 1) / A.S;
        chunk = (chunk + 3) & ~(int64_t)3;
        const int64_t row0 = min(A.n, (int64_t)b * chunk);
        const int64_t row1 = min(A.n, row0 + chunk);
        const int64_t nqa = (row1 - row0 + 3) >> 2;  // quads, the last one possibly partial
        const int64_t steps = (nqa + RT_PT * RT_QPT - 1) / (RT_PT * RT_QPT);
        const int cb = Q * (b % A.R);  // consumer of partition 0
        const bool vec = ((((uintptr_t)A.keys) | ((uintptr_t)A.vals)) & 15) == 0;
        const uint32_t qcnt_s = (uint32_t)__cvta_generic_to_shared(qcnt);
        auto load = [&](int64_t qi, QuadT<DT> &q, uint32_t &in) {
            in = 0;
            if (qi >= nqa) { q = QuadT<DT>{}; return; }
            const int64_t r = row0 + 4 * qi;
            const int c = (int)min((int64_t)4, row1 - r);
            if (c == 4) load_quad_rt<DT>(A.keys, A.vals, r, q, vec);
            else load_partial<DT>(A.keys, A.vals, r, c, q);
            in = (1u << c) - 1u;
        };
        QuadT<DT> nxt[RT_QPT];
        uint32_t nin[RT_QPT];
#pragma unroll
        for (int i = 0; i < RT_QPT; ++i) load(i * RT_PT + ptid, nxt[i], nin[i]);
        bool aborted = false;
        for (int64_t s = 0; s < steps; ++s) {
            QuadT<DT> q[RT_QPT];
            uint32_t in[RT_QPT];
#pragma unroll
            for (int i = 0; i < RT_QPT; ++i) {
                q[i] = nxt[i];
                in[i] = nin[i];
                if (!RT_LATE_LOAD) load((s + 1) * RT_PT * RT_QPT + i * RT_PT + ptid, nxt[i], nin[i]);
            }
            if (RT_L2PF && vec && lane == 0) {
#pragma unroll
                for (int i = 0; i < RT_QPT; ++i) {
                    const int64_t qp = (s + 2) * RT_PT * RT_QPT + i * RT_PT + warp * 32;
                    if (qp + 32 <= nqa && row0 + 4 * (qp + 32) <= row1) {
                        const int64_t r = row0 + 4 * qp;
                        l2_prefetch(A.keys + r, 128 * 4);
                        l2_prefetch(A.vals + r, 128 * (uint32_t)sizeof(V));
                    }
                }
            }
            RT_T0();
            // classify: EKEY, heavy (deposited here), or partition qq / local key;
            // rank within (tile, partition) by one shared atomic per row
            int qq[RT_QPT][4];
            uint32_t rk[RT_QPT][4];
            int32_t lk[RT_QPT][4];
#pragma unroll
            for (int i = 0; i < RT_QPT; ++i) {
                uint32_t hin = 0;
                int hcol[4], hs[4];
                V hv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int32_t k = kq(q[i].k, u);
                    qq[i][u] = -1;
                    rk[i][u] = 0;
                    lk[i][u] = 0;
                    hcol[u] = RT_NH * 32 + lane;
                    hs[u] = RT_NH * 32 + lane;
                    hv[u] = q[i].v(u);
                    if (!((in[i] >> u) & 1u)) continue;
                    if ((uint32_t)k >= (uint32_t)A.G) { flags |= FLAG_EKEY; continue; }
                    const int h = nh ? heavy_of(hhash, k) : -1;
                    if (h >= 0) { hin |= 1u << u; hcol[u] = 32 * h + lane; continue; }
                    const uint32_t l_ = Q > 1 ? __umulhi((uint32_t)k, A.M) : (uint32_t)k;
                    lk[i][u] = (int32_t)l_;
                    qq[i][u] = k - (int)l_ * Q;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (qq[i][u] >= 0) rk[i][u] = atom_add_shared(qcnt_s + 4u * (uint32_t)qq[i][u], 1u);
                if (__any_sync(0xffffffffu, hin != 0u))
                    deposit(hbase, hws, hcol, hs, hv, hin, gid_heavy, mark_heavy);
            }
            pbar();
            RT_T(1);
            // thread t: reserve partition t's run in its consumer's ring and
            // check for room (qst 2: writable now, 0: not yet, 1: no rows).  A
            // reservation is held until it is written, and the consumer cannot
            // pass an unwritten one, so a run is reserved only while the ring
            // looks at most half full (by this thread's last reservation end,
            // which trails the ring's tail by up to a tile of every producer):
            // otherwise producers that reserve ahead of the room would keep the
            // ring full and the consumer would advance one handshake at a time
            bool notready = false, pend = false;
            int v = 0;
            if (ptid < Q) {
                v = qcnt[ptid];
                qcnt[ptid] = 0;  // (the next tile's ranks start after two barriers)
                pend = v > 0;
                if (!pend) qst[ptid] = 1;
            }
            auto try_reserve = [&]() {
                const size_t hq = (size_t)(cb + ptid) * RT_PADW;
                const unsigned long long cap = RT_RING / 2;
                if (lend[ptid] > hcache[ptid] + cap) {
                    hcache[ptid] = ld_vol_u64(A.head + hq);
                    if (lend[ptid] > hcache[ptid] + cap) return;
                }
                const unsigned long long pos = atomicAdd(&A.tail[hq], (unsigned long long)v);
                qpos[ptid] = pos;
                qpos32[ptid] = (uint32_t)pos;
                const unsigned long long end = pos + (unsigned long long)v;
                lend[ptid] = end;
                int st_ = 2;
                if (end > (unsigned long long)RT_RING) {
                    const unsigned long long need = end - RT_RING;
                    if (hcache[ptid] < need) hcache[ptid] = ld_vol_u64(A.head + hq);
                    if (hcache[ptid] < need) { st_ = 0; qoff[ptid] = v; }  // (qoff: the run length, for rechecks)
                }
                qst[ptid] = st_;
                notready = st_ == 0;
                pend = false;
            };
            if (RT_DIAG == 1) { pend = false; if (ptid < Q) qst[ptid] = 1; }
            if (pend) try_reserve();
            bool all_ready = true;
            if (pbar_count(pend || notready) != 0) {  // (rare) deferred reservations or rings without room
                RT_C(8);
                long long rs = 0;
                while (pbar_count(pend) != 0) {
                    RT_C(9);
                    bool ab = false;
                    if (ptid == 0) ab = ++rs > RT_SPIN || ld_vol_i32(A.ctrl + RC_ABORT) != 0;
                    __nanosleep(128);
                    if (pend) try_reserve();
                    if (pbar_count(ab)) { aborted = true; break; }
                }
                all_ready = pbar_count(notready) == 0;
            }
            if (aborted) break;
            if (RT_LATE_LOAD) {
#pragma unroll
                for (int i = 0; i < RT_QPT; ++i) load((s + 1) * RT_PT * RT_QPT + i * RT_PT + ptid, nxt[i], nin[i]);
            }
            RT_T(4);
            // write every row whose run has room, straight from registers;
            // repeat until all are written.  A row's slot and lap tag need
            // only the low 32 bits of its position.
            auto put = [&](V val, int p, uint32_t r_, int32_t l_) {
                const uint32_t pos = qpos32[p] + r_;
                const uint32_t hw = (~(pos << (31 - RT_RING_LOG)) & 0x80000000u);  // lap tag, bit 31 of a high word
                const uint32_t idx = ((uint32_t)(cb + p) << RT_RING_LOG) | (pos & (RT_RING - 1));
                unsigned long long *dst = A.ring + (size_t)idx * RT_W<DT>;
                const unsigned long long kw = (unsigned long long)(hw | (uint32_t)l_) << 32;
                if constexpr (DT == 1) {
                    const unsigned long long vb = (unsigned long long)__double_as_longlong((double)val);
                    st_v2_u64(dst, kw | (vb & 0xffffffffull), ((unsigned long long)hw << 32) | (vb >> 32));
                } else {
                    st_u64(dst, kw | __float_as_uint((float)val));
                }
            };
            uint32_t left = 0;  // bit 4 i + u: row not written yet
            if (RT_DIAG == 1) {
            } else if (all_ready) {  // (producer-uniform) the common case: every run has room
#pragma unroll
                for (int i = 0; i < RT_QPT; ++i)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (qq[i][u] >= 0) put(q[i].v(u), qq[i][u], rk[i][u], lk[i][u]);
            } else {
#pragma unroll
                for (int i = 0; i < RT_QPT; ++i)
#pragma unroll
                    for (int u = 0; u < 4; ++u) left |= qq[i][u] >= 0 ? 1u << (4 * i + u) : 0u;
            }
            long long spins = 0;
            while (!all_ready) {
#pragma unroll
                for (int i = 0; i < RT_QPT; ++i)
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (!((left >> (4 * i + u)) & 1u) || qst[qq[i][u]] != 2) continue;
                        left &= ~(1u << (4 * i + u));
                        put(q[i].v(u), qq[i][u], rk[i][u], lk[i][u]);
                    }
                if (pbar_count(left != 0u) == 0) break;
                RT_C(10);
                // some runs had no room: wait, re-check them
                bool ab = false;
                if (ptid == 0) ab = ++spins > RT_SPIN || ld_vol_i32(A.ctrl + RC_ABORT) != 0;
                __nanosleep(64);
                if (ptid < Q && qst[ptid] == 0) {
                    const unsigned long long need = qpos[ptid] + (unsigned long long)qoff[ptid] - RT_RING;
                    hcache[ptid] = ld_vol_u64(A.head + (size_t)(cb + ptid) * RT_PADW);
                    if (hcache[ptid] >= need) qst[ptid] = 3;  // writable from the next pass
                }
                if (pbar_count(ab)) { aborted = true; break; }
                if (ptid < Q && qst[ptid] == 3) qst[ptid] = 2;
                pbar();
            }
            RT_T(6);
            if (aborted) break;  // (producer-uniform: a barrier count)
        }
        __threadfence();
        pbar();
        if (ptid == 0) {
            if (aborted) { atomicExch(A.ctrl + RC_ABORT, 1); flags |= FLAG_ESTALL; }
            atomicAdd(A.ctrl + RC_DONE, 1);
        }
    } else if (cons) {
        // ---------------- consumer ----------------
        const int cw = warp - RT_PW;
        const unsigned long long *rg = A.ring + (size_t)b * RT_RING * RT_W<DT>;
        const unsigned long long *tailp = A.tail + (size_t)b * RT_PADW;
        const int sinkc = gq - 1;
        unsigned long long tl = 0;       // last tail seen
        unsigned long long tfin = ~0ull; // final tail once known
        long long spins = 0;
        bool stalled = false;
        long long mn_seen = 0;  // a lower bound of the slowest warp's next batch
        for (long long kbat = cw;; kbat += RT_CWN) {
            // at most RT_LEAD batches ahead of the slowest consumer warp (the
            // shared progress words are read only near the bound)
            while (kbat >= mn_seen + RT_LEAD) {
                int mn = 0x7fffffff;
#pragma unroll
                for (int w = 0; w < RT_CWN; ++w) mn = min(mn, *(volatile int *)&s_cprog[w]);
                mn_seen = mn;
                if (kbat < (long long)mn + RT_LEAD) break;
                if (++spins > RT_SPIN) { stalled = true; break; }
                __nanosleep(64);
            }
            if (stalled) break;
            RT_T0();
            const unsigned long long p0 = (unsigned long long)kbat * RT_BATCH;
            const unsigned long long pl = p0 + 4 * lane;
            const uint32_t slot = (uint32_t)(pl & (RT_RING - 1));
            const unsigned long long tag = lap_tag(p0);
            unsigned long long wd[4][RT_W<DT>];
            uint32_t in = 0;
            bool past = false;  // the whole batch lies at or past the final tail (warp-uniform)
            // cheap probe first (lane 31, one word, exponential backoff) so that
            // idle consumers do not flood L2: wait until the batch's last row
            // is reserved and written, or the stream is over
            {
                unsigned ns_ = 32;
                for (int it = 0; it < 48; ++it) {
                    int go = 0;
                    unsigned long long t1 = tl;
                    if (lane == 31) {
                        if (p0 + RT_BATCH > t1) t1 = ld_vol_u64(tailp);
                        if (p0 + RT_BATCH <= t1) {
                            const unsigned long long w = ld_vol_u64(rg + (size_t)(slot + 3) * RT_W<DT> + RT_W<DT> - 1);
                            go = (w & (1ull << 63)) == tag;
                        } else {
                            go = ld_vol_i32(A.ctrl + RC_DONE) == A.S;
                        }
                    }
                    tl = __shfl_sync(0xffffffffu, t1, 31);
                    if (__shfl_sync(0xffffffffu, go, 31)) break;
                    RT_C(11);
                    __nanosleep(ns_);
                    ns_ = min(ns_ * 2, 512u);
                }
            }
            unsigned bo = 64;
            for (;;) {
#pragma unroll
                for (int u = 0; u < 4 * RT_W<DT>; u += 2)
                    ld_vol_v2_u64(rg + (size_t)slot * RT_W<DT> + u, wd[u / RT_W<DT>][u % RT_W<DT>],
                                  wd[(u + 1) / RT_W<DT>][(u + 1) % RT_W<DT>]);
                // tail and end-of-stream decisions are read by lane 0 and broadcast
                unsigned long long t0 = tl;
                if (lane == 0 && p0 + RT_BATCH > tl && tl < tfin) t0 = ld_vol_u64(tailp);
                tl = __shfl_sync(0xffffffffu, t0, 0);
                const unsigned long long lim_ = min(tl, tfin);
                uint32_t rdy = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    bool ok = pl + u < lim_;
#pragma unroll
                    for (int x = 0; x < RT_W<DT>; ++x) ok = ok && (wd[u][x] & (1ull << 63)) == tag;
                    rdy |= ok ? 1u << u : 0u;
                }
                // rows at or past the final tail never come
                uint32_t gone = 0;
                if (tfin != ~0ull)
#pragma unroll
                    for (int u = 0; u < 4; ++u) gone |= pl + u >= tfin ? 1u << u : 0u;
                if (__all_sync(0xffffffffu, (rdy | gone) == 0xFu)) {
                    in = rdy;
                    past = tfin != ~0ull && p0 >= tfin;
                    break;
                }
                if (tfin == ~0ull) {
                    int dn = 0;
                    if (lane == 0) dn = ld_vol_i32(A.ctrl + RC_DONE) == A.S;
                    if (__shfl_sync(0xffffffffu, dn, 0)) {
                        __threadfence();
                        unsigned long long tf = 0;
                        if (lane == 0) tf = ld_vol_u64(tailp);
                        tfin = __shfl_sync(0xffffffffu, tf, 0);
                        tl = tfin;
                        continue;
                    }
                }
                int ab = 0;
                if (lane == 0) ab = ld_vol_i32(A.ctrl + RC_ABORT);
                if (++spins > RT_SPIN || __shfl_sync(0xffffffffu, ab, 0)) {
                    stalled = true;
                    break;
                }
                __nanosleep(bo);
                bo = min(bo * 2, 256u);
            }
            if (stalled) break;
            RT_T(2);
            if (past) break;
            V v[4];
            int cl[4];
            const int sink[4] = {sinkc, sinkc, sinkc, sinkc};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool iu = (in >> u) & 1u;
                cl[u] = iu ? (int)((uint32_t)(wd[u][0] >> 32) & 0x7fffffffu) : sinkc;
                if constexpr (DT == 1)
                    v[u] = iu ? __longlong_as_double((long long)(((wd[u][RT_W<DT> - 1] & 0xffffffffull) << 32) |
                                                                 (wd[u][0] & 0xffffffffull)))
                              : 0.0;
                else
                    v[u] = iu ? __uint_as_float((uint32_t)wd[u][0]) : 0.0f;
            }
            deposit(cbase, cws, cl, sink, v, in, gid_local, mark_local);
            RT_T(3);
            __syncwarp();
            if (lane == 0) {
                s_cprog[cw] = (int)(kbat + RT_CWN);
                int mn = 0x7fffffff;
#pragma unroll
                for (int w = 0; w < RT_CWN; ++w) mn = min(mn, *(volatile int *)&s_cprog[w]);
                const unsigned long long h = (unsigned long long)mn * RT_BATCH;
                if (h >= s_pub + RT_PUB) {
                    s_pub = h;
                    atomicMax(A.head + (size_t)b * RT_PADW, h);
                }
            }
        }
        if (lane == 0) {
            s_cprog[cw] = 0x7fffffff - RT_LEAD;  // no longer holds the others back
            if (stalled) {  // release every waiting producer: the result is void (FLAG_ESTALL)
                flags |= FLAG_ESTALL;
                atomicExch(A.ctrl + RC_ABORT, 1);
                atomicMax(A.head + (size_t)b * RT_PADW, ~0ull >> 1);
            }
        }
    }
    __syncthreads();
    // publish the table: every counter at its absolute level, the tops reached
    if (cons)
        for (int j = tid; j < gb; j += RT_TPB) {
            const int64_t g = (int64_t)j * Q + qown;
#pragma unroll
            for (int lv = 0; lv < NL; ++lv) {
                int64_t T = 0;
#pragma unroll
                for (int h = 0; h < LIMBS; ++h) {
                    const int w = lv * LIMBS + h;
                    T += counter_part<DT>(w, cnt[(size_t)w * gq + j]);
                }
                if (kb - lv >= 1 - K) slot_add<DT, K>(A.slots, g, kb - lv, T);
            }
            const uint32_t t = (topb[j >> 4] >> ((j & 15) * 2)) & 3u;
            const int top = (t & 2u) ? kb : (t & 1u) ? kb - 1 : 0;
            if (top > 0) atomicMax(&A.kglob[g], top);
        }
    for (int i = tid; i < nh * CWB; i += RT_TPB) {
        const int h = i / CWB, w = i - h * CWB;
        int64_t T = 0;
        for (int l = 0; l < 32; ++l) T += counter_part<DT>(w, hcnt[(size_t)w * RT_HCOLS + 32 * h + l]);
        if (kb - w / LIMBS >= 1 - K) slot_add<DT, K>(A.slots, A.ctrl[RC_HKEY + h], kb - w / LIMBS, T);
    }
    for (int h = tid; h < nh; h += RT_TPB) {
        const uint32_t t = htop[h];
        const int top = (t & 2u) ? kb : (t & 1u) ? kb - 1 : 0;
        if (top > 0) atomicMax(&A.kglob[A.ctrl[RC_HKEY + h]], top);
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0 && flags) atomicOr(A.status, flags);
#if RT_PROF
    if (tid == 0 || tid == RT_PT)  // producer thread 0: phases 1, 4, 5, 6; consumer warp 0 lane 0: 2, 3
        for (int i = 1; i < 12; ++i) atomicAdd(&g_rt_prof[i], (unsigned long long)rt_acc[i]);
    if (tid == 0) atomicAdd(&g_rt_prof[0], 1ull);
#endif
}

template <int DT, int K, int XB>
struct RtPlan {
    int Q, R, gq;
    size_t smem;
};

// partitions and table size for G groups (Q = 0: does not apply)
template <int DT, int K, int XB>
RtPlan<DT, K, XB> rt_plan(int32_t G) {
    using Geo = RtGeo<DT, K, XB>;
    RtPlan<DT, K, XB> p{};
    const int S = device_props().sms;
    const size_t budget = (size_t)device_props().smem_optin - 1024;
    if (Geo::bytes(8) > budget) return p;
    // largest gq (multiple of 4) that fits
    int lo = 8, hi = 1 << 20;
    while (hi - lo > 4) {
        const int mid = ((lo + hi) / 2) & ~3;
        if (Geo::bytes(mid) <= budget) lo = mid; else hi = mid;
    }
    const int cap = lo - 1;  // local groups (one column is the sink)
    const int qmin = (int)(((int64_t)G + cap - 1) / cap);
    if (qmin > std::min(S, RT_QMAX)) return p;
    p.R = S / qmin;
    p.Q = std::min(S / p.R, RT_QMAX);
    if ((unsigned long long)G * (unsigned long long)p.Q >= 0x100000000ull) { p.Q = 0; return p; }
    const int gbmax = (int)(((int64_t)G + p.Q - 1) / p.Q);
    p.gq = (gbmax + 1 + 3) & ~3;
    p.smem = Geo::bytes(p.gq);
    return p;
}

struct RtWs {
    int32_t *kglob;
    unsigned long long *slots;
    int32_t *ctrl;
    unsigned long long *tail, *head;
    unsigned long long *ring;
    size_t zero_bytes;
    size_t bytes;
};

template <int DT, int K>
RtWs rt_carve(void *ws, int32_t G) {
    using V = typename Fmt<DT>::V;
    constexpr int NS = Fmt<DT>::KMAX + K;
    const int S = device_props().sms;
    RtWs w{};
    char *b = (char *)ws;
    size_t o = 0;
    auto take = [&](size_t bytes) { char *p = b + o; o += (bytes + 255) / 256 * 256; return p; };
    w.kglob = (int32_t *)take(4 * (size_t)G);
    w.slots = (unsigned long long *)take(16 * (size_t)G * NS);
    w.ctrl = (int32_t *)take(4 * RC_WORDS);
    w.tail = (unsigned long long *)take(8 * (size_t)S * RT_PADW);
    w.head = (unsigned long long *)take(8 * (size_t)S * RT_PADW);
    w.ring = (unsigned long long *)take(8 * (size_t)S * RT_RING * RT_W<DT>);
    w.zero_bytes = o;
    w.bytes = o;
    return w;
}

template <int DT, int K, int XB>
int launch_route_xb(const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws, size_t ws_bytes,
                    const RtPlan<DT, K, XB> &pl, int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out,
                    uint32_t *status, cudaStream_t st, int *launches) {
    using V = typename Fmt<DT>::V;
    const int S = device_props().sms;
    RtWs w = rt_carve<DT, K>(ws, G);
    if (w.bytes > ws_bytes) return -1;
    static thread_local size_t conf_r = 0, conf_s = 0;
    if (conf_r < pl.smem) {
        if (cudaFuncSetAttribute(k_route<DT, K, XB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem) !=
            cudaSuccess)
            return -2;
        conf_r = pl.smem;
    }
    const size_t sm_s = sizeof(int2) * RT_SHASH;
    if (conf_s < sm_s) {
        if (cudaFuncSetAttribute(k_rt_sample<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_s) !=
            cudaSuccess)
            return -2;
        conf_s = sm_s;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_route<DT, K, XB>, RT_TPB, pl.smem);
    if (per_sm < 1) return -1;
    if (cudaMemsetAsync(ws, 0, w.zero_bytes, st) != cudaSuccess) return -2;
    if (n > 0) {
        int tok = trace_begin(st);
        k_rt_sample<DT><<<1, 1024, sm_s, st>>>(keys, (const V *)vals, n, G, XB, w.ctrl);
        ++*launches;
        trace_end(tok, "route_sample", st);
        RtArgs<DT> A{};
        A.keys = keys;
        A.vals = (const V *)vals;
        A.n = n;
        A.G = G;
        A.Q = pl.Q;
        A.R = pl.R;
        A.S = S;
        A.M = pl.Q > 1 ? (uint32_t)((0x100000000ull + (unsigned long long)pl.Q - 1) / (unsigned long long)pl.Q) : 0u;
        A.gq = pl.gq;
        A.ring = w.ring;
        A.tail = w.tail;
        A.head = w.head;
        A.ctrl = w.ctrl;
        A.kglob = w.kglob;
        A.slots = w.slots;
        A.status = status;
        void *args[] = {&A};
        tok = trace_begin(st);
        const cudaError_t e = cudaLaunchCooperativeKernel((const void *)k_route<DT, K, XB>, dim3(S), dim3(RT_TPB),
                                                          args, pl.smem, st);
        ++*launches;
        trace_end(tok, "route", st);
        if (e == cudaErrorCooperativeLaunchTooLarge) {  // not every SM free (e.g. a concurrent stream):
            (void)cudaGetLastError();                    // the sweep runs instead (it re-zeroes its own workspace)
            return -1;
        }
        if (e != cudaSuccess) return -2;
    }
    if (!out && !acc_k) return 0;  // deposit only (the split form reads the slot table)
    return launch_fold(DT, K, G, w.kglob, w.slots, merge, acc_k, acc_C, acc_D, out, status, st, launches);
}

int g_route_mode = 0;  // 0 off (default: measured slower than the sweep), 1 on where it applies

template <int DT, int K>
int launch_route_t(const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws, size_t ws_bytes, int merge,
                   int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out, uint32_t *status, cudaStream_t st,
                   int *launches) {
    // the band of two window tops when its table still fits, else one
    const auto p1 = rt_plan<DT, K, 1>(G);
    if (p1.Q > 0)
        return launch_route_xb<DT, K, 1>(keys, vals, n, G, ws, ws_bytes, p1, merge, acc_k, acc_C, acc_D, out, status,
                                         st, launches);
    const auto p0 = rt_plan<DT, K, 0>(G);
    if (p0.Q > 0)
        return launch_route_xb<DT, K, 0>(keys, vals, n, G, ws, ws_bytes, p0, merge, acc_k, acc_C, acc_D, out, status,
                                         st, launches);
    return -1;
}

template <int DT, int K>
size_t route_ws_t(int32_t G) {
    if (rt_plan<DT, K, 1>(G).Q <= 0 && rt_plan<DT, K, 0>(G).Q <= 0) return 0;
    return rt_carve<DT, K>(nullptr, G).bytes;
}

}  // namespace

void set_route_mode(int m) { g_route_mode = (m == 0) ? 0 : 1; }
int route_mode() { return g_route_mode; }

size_t route_workspace_bytes(int32_t G, int K, int DT) {
#define RWB(dt, k) \
    if (DT == dt && K == k) return route_ws_t<dt, k>(G);
    RWB(1, 1) RWB(1, 2) RWB(1, 3) RWB(1, 4) RWB(0, 1) RWB(0, 2) RWB(0, 3) RWB(0, 4)
#undef RWB
    return 0;
}

int launch_route(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws,
                 size_t ws_bytes, int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out,
                 uint32_t *status, cudaStream_t st, int *launches) {
    if (!g_route_mode) return -1;
#define RTL(dt, k)          \
    if (DT == dt && K == k) \
        return launch_route_t<dt, k>(keys, vals, n, G, ws, ws_bytes, merge, acc_k, acc_C, acc_D, out, status, st, launches);
    RTL(1, 1) RTL(1, 2) RTL(1, 3) RTL(1, 4) RTL(0, 1) RTL(0, 2) RTL(0, 3) RTL(0, 4)
#undef RTL
    return -1;
}

}  // namespace repro

#if RT_PROF
// debug builds: summed cycles per phase of k_route since the last read
// [0] blocks, producer thread 0: [1] classify+rank [4] scan+reserve [5] stage
// [6] write passes; consumer warp 0: [2] waiting for rows [3] deposit
extern "C" int repro_debug_route_prof(unsigned long long *out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, repro::g_rt_prof, sizeof(unsigned long long) * 12);
    const unsigned long long z[16] = {};
    cudaMemcpyToSymbol(repro::g_rt_prof, z, sizeof(z));
    return 0;
}
#endif
