// k_sweep.cu -- the high-cardinality GroupBy:
// PartitionAndAggregate (Alg. 4) for group counts above
// the on-chip table's capacity, in at most two passes over the rows' bytes
// plus one over the keys.
//
// Groups are split into P <= 256 partitions of Gp = 2^gbits consecutive keys
// (Gp sized so that one partition's table fits on chip: F = f^d with d = 1,
// PAPER.md:1054-1058).
//   1. k_sw_sample  8192 evenly spaced keys; a partition holding >= 1/8 of
//                   them and >= 4x its uniform share is HOT (skew, e.g.
//                   Zipf's head).
//   2. k_sweep_hot  (hot partition only) one pass over the rows: hot rows are
//                   deposited on chip right away (table_core.cuh; the heavy
//                   partition never goes back to HBM), the others are
//                   compacted, coalesced per warp, into a contiguous buffer.
//   3. k_sw_hist    per cold block: rows per partition (the keys only).
//   4. k_sw_scan    per (partition, block): exclusive scan -> every block's
//                   destination range in every partition; partitions start on
//                   whole quads (the gap is padded); accumulate work items.
//   5. k_sweep_cold per tile: rank rows by partition (shared atomics), stage
//                   them in partition order, write each partition's run to
//                   the block's running position in that partition.  Runs of
//                   consecutive tiles abut, so their partial sectors are
//                   completed in L2 before write-back.
//   6. k_sweep_acc  persistent blocks pull work items (row ranges of one
//                   partition) and run the on-chip table over them.
// Plans of 2 .. SW_REP_MAXP partitions skip 1-6 for the REPLICATED-READ form
// (k_sweep_hot<REP>): P blocks stream each row chunk at the same pace, each
// depositing one partition's rows on chip; the later readers hit L2, so HBM
// sees the rows once (12 B per binary64 row) and nothing is written back.
// All tables publish into the absolute-level slot table (kglob, slots) that
// k_fold (k_state.cu) turns into canonical states and Eq. 1 read-outs.  Each
// group lives in exactly one partition; the order of rows inside a partition
// is irrelevant (the accumulator is associative).
//
// HBM traffic per binary64 row: no hot partition: keys 4 (hist) + 12 read +
// 12 written (scatter) + 12 read (accumulate) = 40 B; with a hot partition
// holding a share h of the rows: 12 + (1 - h) (12 + 4 + 24 + 12) B.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"
#include "table_core.cuh"

#include <algorithm>
#include <cstdlib>

namespace repro {

namespace {

constexpr int SW_TPB = 512;            // accumulate blocks (one per SM: the table)
constexpr int SW_HTPB = 512;           // hot-partition pass (one block per SM: the hot table)
#ifndef SW_STPB
#define SW_STPB 256   // scatter block size
#endif
#ifndef SW_HU
#define SW_HU 16      // 16-byte key vectors in flight per histogram thread (4: 0.29 ms, 8: 0.24, 16: 0.21 at 2^28 keys)
#endif
#ifndef SW_HQ
#define SW_HQ 1       // hot pass: quads per thread per step (issue-bound: 2 and 4 measured slower)
#endif
#ifndef SW_L2PF
#define SW_L2PF 0     // scatter / accumulate: lane 0 of each warp bulk-prefetches its rows two steps ahead into L2
#endif
#ifndef SW_SQPT
#define SW_SQPT 2     // quads per thread per scatter tile
#endif
#ifndef SW_BAL
#define SW_BAL 1      // accumulate: equal row ranges per SM cut at partition bounds (0: 2^19-row items from a queue)
#endif
#ifndef SW_PUBROWS
#define SW_PUBROWS 131072  // SW_BAL cost of one table clear + publish in rows (~60 us at G_p = 4096, binary64 K = 3)
#endif
#ifndef SW_MRANK
#define SW_MRANK 8    // scatter ranks by warp match + one atomic per distinct partition up to this many partitions
#endif                // (P = 4: 1.744 -> 1.542 ms; P = 16: 1.617 -> 1.743; P = 256: 2.30 -> 3.07 -- one atomic per row)
#ifndef SW_REP_MAXP
#define SW_REP_MAXP 3  // plans of 2 .. SW_REP_MAXP partitions take the replicated-read form (k_sweep_hot<REP>):
                       // 2^28 rows, scatter form -> replicated: binary64 K=3 P=2 2.67 -> 1.80 ms, P=3 2.67 -> 2.57, P=4 2.68 -> 3.39;
                       // binary32 K=2 P=2 2.15 -> 1.18, P=3 2.19 -> 1.71; binary64 K=2 P=3 2.52 -> 2.07
#endif
#ifndef SW_CBPS64
#define SW_CBPS64 2   // scatter blocks per SM, binary64 (shared memory: stage + carry)
#endif
#ifndef SW_CBPS32
#define SW_CBPS32 3   // the same, binary32
#endif
constexpr int SW_CTPB = 256;           // histogram blocks
constexpr int SW_CTILE = 4 * SW_SQPT * SW_STPB;  // rows per scatter tile
constexpr int SW_RUN = 8;              // rows per written run unit: 32-byte sectors of keys and values
// histogram / scatter blocks per SM (one histogram block per scatter block)
template <int DT>
constexpr int sw_cbps() { return DT == 1 ? SW_CBPS64 : SW_CBPS32; }
constexpr int SW_PMAX = 256;           // partitions of one sweep (<= SW_CTPB: one thread per partition)
constexpr int SW_SAMPLE = 8192;
constexpr int64_t SW_IROWS = 1 << 19;  // rows per accumulate work item (whole quads)
constexpr int SW_TABLE_MAX = 200 * 1024;  // accumulate table (band layout, XB = 1)
// control words: [0] work items, [1] queue head, [3] hot partition, [4] rows
// in the compacted cold buffer, [5] heavy groups of the hot partition,
// [8 .. 8 + TAB_HMAX) their local keys
constexpr int SW_CTRL = 8 + TAB_HMAX;
constexpr int32_t SW_PAD = -1;         // key of a padding row (partition starts on whole quads)

template <int DT, int K>
int sw_gbits() {  // largest power-of-two partition whose table fits SW_TABLE_MAX
    int b = 13;
    while (b > 8 && TabGeom<DT, K, 1>::bytes(1 << b) > SW_TABLE_MAX) --b;
    return b;
}

// one launch, bracketed by the per-kernel timing events when enabled
template <class Fn>
int traced(const char *name, cudaStream_t st, int *launches, Fn &&fn) {
    const int tok = trace_begin(st);
    fn();
    ++*launches;
    trace_end(tok, name, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

struct SwPlan {
    int gbits, Gp, P, grid, cgrid;  // grid: hot pass blocks (1 per SM); cgrid: histogram / scatter blocks
    int64_t rows_cap, max_items;    // partitioned buffer rows; work items
};

template <int DT, int K>
SwPlan sw_plan(int64_t n, int32_t G) {
    SwPlan pl{};
    pl.gbits = sw_gbits<DT, K>();
    pl.Gp = 1 << pl.gbits;
    pl.P = (int)(((int64_t)G + pl.Gp - 1) >> pl.gbits);
    pl.grid = device_props().sms;
    pl.cgrid = sw_cbps<DT>() * device_props().sms;
    // every (scatter block, partition) range is padded to whole run units
    pl.rows_cap = n + (int64_t)SW_RUN * pl.cgrid * pl.P + SW_RUN;
    pl.max_items = SW_BAL ? pl.P + pl.grid + 1 : pl.P + (pl.rows_cap + SW_IROWS - 1) / SW_IROWS + 1;
    return pl;
}

// scatter stage: the tile's rows + every partition's carried rows (< SW_RUN
// each), in partition order
constexpr int SW_STAGE = SW_CTILE + (SW_RUN - 1) * SW_PMAX;
template <int DT, typename DstT>
size_t sw_smem_cold() {
    using V = typename Fmt<DT>::V;
    return (size_t)SW_STAGE * (4 + sizeof(V) + sizeof(DstT)) + (size_t)SW_PMAX * SW_RUN * (4 + sizeof(V)) +
           (size_t)SW_PMAX * (8 + 4 * 4);
}

struct SwWs {
    int32_t *kglob;
    unsigned long long *slots;
    int32_t *ctrl;
    int64_t *hcnt;      // [grid] cold rows each hot-pass block compacted
    size_t zero_bytes;  // kglob .. hcnt (one memset)
    int32_t *bkeys;     // compacted cold rows (hot partition present): block b's at [b chunk, b chunk + hcnt[b])
    void *bvals;
    int32_t *pkeys;     // partitioned rows (local keys; SW_PAD in the gaps)
    void *pvals;
    int64_t *cnt;       // [cgrid][P] rows per (block, partition), then destination bases
    int64_t *pstart;    // [P + 1] first row of each partition
    int64_t *items;     // [max_items][3] partition, first row, end row
    int32_t *bfirst;    // [grid + 1] first item of each accumulate block (SW_BAL)
    size_t bytes;
};

constexpr size_t SWA = 256;
inline size_t swal(size_t x) { return (x + SWA - 1) / SWA * SWA; }

template <int DT, int K>
SwWs sw_carve(void *ws, int64_t n, int32_t G, const SwPlan &pl) {
    using V = typename Fmt<DT>::V;
    constexpr int NS = Fmt<DT>::KMAX + K;
    SwWs w{};
    char *b = (char *)ws;
    size_t o = 0;
    auto take = [&](size_t bytes) { char *p = b + o; o += swal(bytes); return p; };
    w.kglob = (int32_t *)take(4 * (size_t)G);
    w.slots = (unsigned long long *)take(16 * (size_t)G * NS);
    w.ctrl = (int32_t *)take(4 * SW_CTRL);
    w.hcnt = (int64_t *)take(8 * (size_t)pl.grid);
    w.zero_bytes = o;
    w.bkeys = (int32_t *)take(4 * (size_t)n + 16);
    w.bvals = take(sizeof(V) * (size_t)n + 16);
    w.pkeys = (int32_t *)take(4 * (size_t)pl.rows_cap);
    w.pvals = take(sizeof(V) * (size_t)pl.rows_cap);
    w.cnt = (int64_t *)take(8 * (size_t)pl.cgrid * pl.P);
    w.pstart = (int64_t *)take(8 * ((size_t)pl.P + 1));
    w.items = (int64_t *)take(24 * (size_t)pl.max_items);
    w.bfirst = (int32_t *)take(4 * ((size_t)pl.grid + 1));
    w.bytes = o;
    return w;
}

// where the hot pass left the compacted cold rows: hot block r's region
// starts at r * hchunk (quad-aligned) and holds hcnt[r] rows
struct ColdSrc {
    const int64_t *hcnt;
    int hgrid;
    int64_t hchunk;
};

// row range of cold block b of nb over the cold input; quad-aligned.  No hot
// partition: the original rows split evenly.  Hot partition: each hot-pass
// region split into nb / hgrid parts (nb >= hgrid: cold grids are a multiple
// of the SM count, hot grids at most the SM count).
__device__ __forceinline__ void cold_range(const int32_t *ctrl, const ColdSrc &cs, int64_t n, int b, int nb,
                                           int64_t &r0, int64_t &r1) {
    int64_t lo = 0, ne = n;
    int parts = nb, part = b;
    if (ctrl[3] >= 0) {
        parts = nb / cs.hgrid;
        const int r = b / parts;
        part = b - r * parts;
        if (r >= cs.hgrid) { r0 = r1 = 0; return; }
        lo = (int64_t)r * cs.hchunk;
        ne = cs.hcnt[r];
    }
    int64_t chunk = (ne + parts - 1) / parts;
    chunk = (chunk + 3) & ~(int64_t)3;
    r0 = lo + min(ne, (int64_t)part * chunk);
    r1 = lo + min(ne, (int64_t)part * chunk + chunk);
}

// 1. hot partition from evenly spaced keys (performance only: any choice
// gives the same bits)
__global__ void __launch_bounds__(1024) k_sw_sample(const int32_t *__restrict__ keys, int64_t n, int32_t G, int gbits,
                                                    int P, int32_t *ctrl) {
    __shared__ int cnt[SW_PMAX];
    __shared__ int hh[1 << 13];  // sampled rows per local key of the hot partition (Gp <= 2^13)
    __shared__ unsigned long long best;
    __shared__ int s_hot;
    const int tid = threadIdx.x;
    for (int i = tid; i < SW_PMAX; i += 1024) cnt[i] = 0;
    for (int i = tid; i < (1 << gbits); i += 1024) hh[i] = 0;
    if (tid == 0) best = 0;
    __syncthreads();
    for (int i = tid; i < SW_SAMPLE; i += 1024) {
        const int64_t r = n * i / SW_SAMPLE;
        if (r < n) {
            const int32_t k = keys[r];
            if ((uint32_t)k < (uint32_t)G) atomicAdd(&cnt[k >> gbits], 1);
        }
    }
    __syncthreads();
    for (int p = tid; p < P; p += 1024)
        if (cnt[p] > 0) atomicMax(&best, ((unsigned long long)cnt[p] << 32) | (unsigned)(SW_PMAX - 1 - p));
    __syncthreads();
    const int samples = (int)min((int64_t)SW_SAMPLE, n);
    if (tid == 0) {
        const int c = (int)(best >> 32);
        // hot: >= 1/8 of the samples AND >= 4x a partition's uniform share
        // (uniform keys over a few partitions are cheaper through the scatter)
        s_hot = (c > 0 && 8 * c >= samples && (int64_t)c * P >= 4 * (int64_t)samples)
                    ? SW_PMAX - 1 - (int)(best & 0xFFFFFFFFu) : -1;
        ctrl[3] = s_hot;
        ctrl[5] = 0;
    }
    __syncthreads();
    const int hot = s_hot;
    if (hot < 0) return;
    // heavy groups of the hot partition: >= 1/512 of the sampled rows each
    for (int i = tid; i < SW_SAMPLE; i += 1024) {
        const int64_t r = n * i / SW_SAMPLE;
        if (r < n) {
            const int32_t k = keys[r];
            if ((uint32_t)k < (uint32_t)G && (k >> gbits) == hot) atomicAdd(&hh[k & ((1 << gbits) - 1)], 1);
        }
    }
    __syncthreads();
    const int thr = max(4, samples / 512);
    for (int i = tid; i < (1 << gbits); i += 1024)
        if (hh[i] >= thr) {
            const int slot = atomicAdd(&ctrl[5], 1);
            if (slot < TAB_HMAX) ctrl[8 + slot] = i;
        }
}

// 2. hot partition present: one pass that deposits the hot rows on chip right
// away (the heavy partition never goes back to HBM) and compacts the other
// rows, coalesced per warp, into a contiguous buffer for 3-5.  Exits at once
// when there is no hot partition.
// REP > 0 (the replicated-read form for plans of 2 .. SW_REP_MAXP partitions):
// no sample, no scatter -- block b streams row chunk b / REP_P and deposits the
// rows of partition b % REP_P only (the others add zeros to the sink columns),
// so the REP_P blocks of one chunk read the same rows at the same pace (the
// later readers hit L2) and nothing is written back to HBM.
template <int DT, int K, bool REP = false>
__global__ void __launch_bounds__(SW_HTPB, 1)
k_sweep_hot(const int32_t *__restrict__ keys, const typename Fmt<DT>::V *__restrict__ vals, int64_t n, int32_t G,
            int gbits, int64_t chunk, int32_t *__restrict__ bkeys, typename Fmt<DT>::V *__restrict__ bvals,
            int32_t *__restrict__ ctrl, int64_t *__restrict__ hcnt, int32_t *__restrict__ kglob,
            unsigned long long *__restrict__ slots, uint32_t *__restrict__ status, int rep_p) {
    using V = typename Fmt<DT>::V;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_mm[TAB_MM];
    __shared__ int s_ccount;  // cold rows compacted by this block (its region starts at row0)
    const int hot = REP ? (int)(blockIdx.x % rep_p) : ctrl[3];
    if (hot < 0) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const int Gp = 1 << gbits;
    const int64_t row0 = (int64_t)(REP ? blockIdx.x / rep_p : blockIdx.x) * chunk;
    const int64_t row1 = min(n, row0 + chunk);
    if (row0 >= row1) return;
    const int nh = REP ? 0 : min(ctrl[5], TAB_HMAX);
    Table<DT, K, SW_HTPB, 0, true, 1> tab(smem, s_mm, min(Gp, G - hot * Gp), (int64_t)hot * Gp, kglob, slots, nh);
    tab.clear();
    if (tid == 0) s_ccount = 0;
    __syncthreads();
    tab.set_heavy(ctrl + 8, nh);
    uint32_t flags = 0;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    auto step = [&](const QuadT<DT> &q, uint32_t in) {
        // branch-free classification: hot rows (hin) go to the table, cold
        // rows (cin) to the compacted buffer, bad keys set EKEY
        uint32_t hin = 0, cin = 0, bad = 0;
        int hk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t k = kq(q.k, u);
            const bool iu = (in >> u) & 1u;
            const bool ok = (uint32_t)k < (uint32_t)G;
            const bool h = ok && (k >> gbits) == hot;
            hin |= (iu && h) ? 1u << u : 0u;
            cin |= (!REP && iu && ok && !h) ? 1u << u : 0u;
            bad |= (iu && !ok) ? 1u : 0u;
            hk[u] = k & (Gp - 1);
        }
        if (bad) flags |= FLAG_EKEY;
        // compaction: one ballot per quad slot; the warp's cold rows of slot u
        // land in consecutive positions (coalesced stores), one shared atomic
        // per warp reserves them in the block's region
        uint32_t m[4] = {0, 0, 0, 0};
        int tot = 0;
        if (!REP) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                m[u] = __ballot_sync(0xffffffffu, (cin >> u) & 1u);
                tot += __popc(m[u]);
            }
        }
        if (!REP && tot) {  // (warp-uniform)
            int base = 0;
            if (lane == 0) base = atomicAdd(&s_ccount, tot);
            base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if ((cin >> u) & 1u) {
                    const int64_t pos = row0 + base + __popc(m[u] & lt);
                    bkeys[pos] = kq(q.k, u);
                    bvals[pos] = q.v(u);
                }
                base += __popc(m[u]);
            }
        }
        QuadT<DT> hq = q;
        hq.k = make_int4(hk[0], hk[1], hk[2], hk[3]);
        tab.quad(hq, hin, flags);
    };
    const int64_t nq = (row1 - row0) >> 2;
    // QH quads per thread per step, the next step's in flight (memory-level
    // parallelism: one block of 512 threads per SM holds the table)
    constexpr int QH = SW_HQ;
    const int64_t steps = (nq + SW_HTPB * QH - 1) / (SW_HTPB * QH);
    QuadT<DT> nxt[QH];
    const bool vec = ((((uintptr_t)keys) | ((uintptr_t)vals)) & 15) == 0;  // (rows r0 are quad multiples)
#pragma unroll
    for (int i = 0; i < QH; ++i)
        if (i * SW_HTPB + tid < nq) load_quad_rt<DT>(keys, vals, row0 + 4 * (int64_t)(i * SW_HTPB + tid), nxt[i], vec);
    for (int64_t s = 0; s < steps; ++s) {
        QuadT<DT> cur[QH];
#pragma unroll
        for (int i = 0; i < QH; ++i) cur[i] = nxt[i];
        const int64_t q0 = s * SW_HTPB * QH + tid;
#pragma unroll
        for (int i = 0; i < QH; ++i) {
            const int64_t qn = q0 + (int64_t)(QH + i) * SW_HTPB;
            if (qn < nq) load_quad_rt<DT>(keys, vals, row0 + 4 * qn, nxt[i], vec);
        }
#pragma unroll
        for (int i = 0; i < QH; ++i) step(cur[i], q0 + (int64_t)i * SW_HTPB < nq ? 0xFu : 0u);
    }
    const int tail = (int)(row1 - row0 - 4 * nq);
    if (tail > 0) {
        QuadT<DT> t;
        load_partial<DT>(keys, vals, row0 + 4 * nq, tid == 0 ? tail : 0, t);
        step(t, tid == 0 ? (1u << tail) - 1u : 0u);
    }
    tab.finish();  // (barriers on both sides: every warp's compaction is done)
    if (!REP && tid == 0) hcnt[blockIdx.x] = s_ccount;
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0 && flags) atomicOr(status, flags);
}

// 3. rows per (cold block, partition); key check on the original rows.
// 16-byte key loads, four in flight per thread.
__global__ void __launch_bounds__(SW_CTPB)
k_sw_hist(const int32_t *__restrict__ keys, const int32_t *__restrict__ bkeys, int64_t n, int32_t G, int gbits,
          int P, const int32_t *__restrict__ ctrl, ColdSrc cs, int64_t *__restrict__ cnt,
          uint32_t *__restrict__ status) {
    __shared__ int h[SW_PMAX];
    const int tid = threadIdx.x;
    const bool compacted = ctrl[3] >= 0;
    const int32_t *k = compacted ? bkeys : keys;
    int64_t r0, r1;
    cold_range(ctrl, cs, n, blockIdx.x, gridDim.x, r0, r1);
    for (int p = tid; p < SW_PMAX; p += SW_CTPB) h[p] = 0;
    __syncthreads();
    uint32_t bad = 0;
    auto one = [&](int32_t key) {
        if ((uint32_t)key < (uint32_t)G) atomicAdd(&h[key >> gbits], 1);
        else bad = FLAG_EKEY;
    };
    int64_t r = r0;
    if ((((uintptr_t)(k + r0)) & 15) == 0) {  // r0 is a multiple of 4; keys may be unaligned
        constexpr int U = SW_HU;
        const int64_t nq = (r1 - r0) >> 2;
        const int4 *kq4 = reinterpret_cast<const int4 *>(k + r0);
        int64_t q = tid;
        for (; q + (U - 1) * SW_CTPB < nq; q += U * SW_CTPB) {
            int4 a[U];
#pragma unroll
            for (int u = 0; u < U; ++u) a[u] = __ldcs(kq4 + q + u * SW_CTPB);
#pragma unroll
            for (int u = 0; u < U; ++u) { one(a[u].x); one(a[u].y); one(a[u].z); one(a[u].w); }
        }
        for (; q < nq; q += SW_CTPB) {
            const int4 a = __ldcs(kq4 + q);
            one(a.x); one(a.y); one(a.z); one(a.w);
        }
        r = r0 + 4 * nq;
    }
    for (r += tid; r < r1; r += SW_CTPB) one(__ldg(k + r));
    __syncthreads();
    for (int p = tid; p < P; p += SW_CTPB) cnt[(size_t)blockIdx.x * P + p] = h[p];
    bad = __reduce_or_sync(0xffffffffu, bad);
    if ((tid & 31) == 0 && bad) atomicOr(status, bad);
}

// 4. destination bases (in place of the counts): every (block, partition)
// range is padded to whole run units of SW_RUN rows, so partitions and block
// ranges start on 32-byte sectors of both columns; work items (single block)
__device__ __forceinline__ int64_t sw_pad(int64_t c) { return (c + SW_RUN - 1) & ~(int64_t)(SW_RUN - 1); }

__global__ void __launch_bounds__(1024)
k_sw_scan(int64_t *__restrict__ cnt, int nb, int P, int64_t *__restrict__ pstart, int32_t *__restrict__ pkeys,
          int64_t *__restrict__ items, int32_t *__restrict__ bfirst, int na, int32_t *__restrict__ ctrl) {
    __shared__ int64_t part[4][SW_PMAX];
    __shared__ int64_t start[SW_PMAX + 1];
    __shared__ int64_t cps[SW_PMAX + 1];  // SW_BAL: cost before each partition
    __shared__ int64_t cuts[1025];        // SW_BAL: first row of each accumulate block (na <= 1024)
    __shared__ int32_t nitm[1025];
    const int tid = threadIdx.x;
    const int p = tid & (SW_PMAX - 1), quarter = tid >> 8;  // 4 threads per partition
    const int b0 = nb * quarter / 4, b1 = nb * (quarter + 1) / 4;
    if (p < P) {
        int64_t t = 0;
#pragma unroll 8
        for (int b = b0; b < b1; ++b) t += sw_pad(cnt[(size_t)b * P + p]);
        part[quarter][p] = t;
    }
    __syncthreads();
    if (tid == 0) {
        int64_t a = 0, it = 0, c = 0;
        for (int q = 0; q < P; ++q) {
            const int64_t tot = part[0][q] + part[1][q] + part[2][q] + part[3][q];
            start[q] = a;
            cps[q] = c;
            if (tot > 0) c += tot + SW_PUBROWS;
            if (!SW_BAL)
                for (int64_t r = 0; r < tot; r += SW_IROWS, ++it) {  // items of whole run units
                    items[3 * it] = q;
                    items[3 * it + 1] = a + r;
                    items[3 * it + 2] = a + min(tot, r + SW_IROWS);
                }
            a += tot;
        }
        start[P] = a;
        cps[P] = c;
        if (!SW_BAL) {
            ctrl[0] = (int32_t)it;
            ctrl[1] = 0;
        }
    }
    if (SW_BAL) {
        // accumulate block b takes rows [cuts[b], cuts[b + 1]) of the
        // partitioned buffer (cuts on whole run units), split where a
        // partition ends (one table clear + publish per partition it
        // touches).  The cuts are equal steps of a cost coordinate in which
        // every non-empty partition costs its rows + SW_PUBROWS; a cut that
        // lands in a partition's publish share snaps to the partition's start.
        __syncthreads();
        const int64_t a = start[P], ctot = cps[P];
        if (tid <= na) {
            int64_t ct = a;
            if (tid < na) {
                const int64_t x = ctot * tid / na;
                if (x < ctot) {
                    int lo = 0, hi = P;  // cps[lo] <= x < cps[hi]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (cps[mid] <= x) lo = mid; else hi = mid;
                    }
                    const int64_t rq = start[lo + 1] - start[lo];
                    ct = start[lo] + (min(rq, max((int64_t)0, x - cps[lo] - SW_PUBROWS)) & ~(int64_t)(SW_RUN - 1));
                }
            }
            cuts[tid] = ct;
        }
        __syncthreads();
        // the non-empty partitions of block tid's range: [qlo, qhi]
        auto part_of = [&](int64_t r) {  // the last partition starting at or before row r (non-empty)
            int lo = 0, hi = P;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (start[mid] <= r) lo = mid; else hi = mid;
            }
            return lo;
        };
        int qlo = 0, qhi = -1;
        if (tid < na && cuts[tid] < cuts[tid + 1]) {
            qlo = part_of(cuts[tid]);
            qhi = part_of(cuts[tid + 1] - 1);
        }
        if (tid < na) {
            int m = 0;
            for (int q = qlo; q <= qhi; ++q) m += start[q + 1] > start[q];
            nitm[tid] = m;
        }
        __syncthreads();
        if (tid == 0) {
            int t = 0;
            for (int b = 0; b < na; ++b) {
                const int m = nitm[b];
                nitm[b] = t;
                t += m;
            }
            nitm[na] = t;
            ctrl[0] = t;
            ctrl[1] = 0;
        }
        __syncthreads();
        if (tid <= na) bfirst[tid] = nitm[tid];
        if (tid < na) {
            int it = nitm[tid];
            for (int q = qlo; q <= qhi; ++q) {
                if (start[q + 1] <= start[q]) continue;
                items[3 * it] = q;
                items[3 * it + 1] = max(cuts[tid], start[q]);
                items[3 * it + 2] = min(cuts[tid + 1], start[q + 1]);
                ++it;
            }
        }
    }
    __syncthreads();
    for (int q = tid; q <= P; q += 1024) pstart[q] = start[q];
    if (p < P) {
        int64_t a = start[p];
        for (int w = 0; w < quarter; ++w) a += part[w][p];
#pragma unroll 8
        for (int b = b0; b < b1; ++b) {
            const int64_t c = cnt[(size_t)b * P + p];
            cnt[(size_t)b * P + p] = a;
            a += sw_pad(c);
        }
    }
}

// 5. the scatter of the cold rows.  Per tile: rank the rows by partition
// (shared atomics); each partition's rows -- the < SW_RUN rows it carried over
// from the previous tile first, then the tile's -- are numbered j = 0 .. T-1;
// rows j < F (F = T rounded down to whole run units of SW_RUN rows: full
// 32-byte sectors of keys and values) are staged, in partition order, with
// their destination (the block's running position in the partition + j), the
// others are carried to the next tile.  The write phase then only reads
// (key, value, destination) per staged row: consecutive threads write
// consecutive rows of a run.  Runs of consecutive tiles abut, and every
// write is a whole, aligned sector, so DRAM never merges partial sectors.  The
// block's last units are padded with SW_PAD rows.  Destinations are DstT:
// 32-bit unless the partitioned buffer holds 2^32 rows or more.
template <int DT, typename DstT, bool MR>
__global__ void __launch_bounds__(SW_STPB, sw_cbps<DT>())
k_sweep_cold(const int32_t *__restrict__ keys, const typename Fmt<DT>::V *__restrict__ vals, int64_t n,
             const int32_t *__restrict__ bkeys, const typename Fmt<DT>::V *__restrict__ bvals, int32_t G, int gbits,
             int P, const int64_t *__restrict__ base, int32_t *__restrict__ pkeys,
             typename Fmt<DT>::V *__restrict__ pvals, const int32_t *__restrict__ ctrl, ColdSrc cs) {
    using V = typename Fmt<DT>::V;
    constexpr int TPB = SW_STPB, NW = TPB / 32, TILE = SW_CTILE, QPT = TILE / (4 * TPB);
    static_assert(TPB >= SW_PMAX, "one thread per partition");
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_wsum[NW];
    __shared__ int s_nw;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Gp = 1 << gbits;
    if (ctrl[3] >= 0) { keys = bkeys; vals = bvals; }
    int64_t row0, row1;
    cold_range(ctrl, cs, n, blockIdx.x, gridDim.x, row0, row1);
    if (row0 >= row1) return;
    // shared memory: stage values | carried values | run | stage keys |
    // stage destinations | carried keys | per-partition counts
    V *tvals = reinterpret_cast<V *>(smem);
    V *cvals = tvals + SW_STAGE;
    int64_t *run = reinterpret_cast<int64_t *>(cvals + SW_PMAX * SW_RUN);  // next destination row per partition
    DstT *tdst = reinterpret_cast<DstT *>(run + SW_PMAX);
    int32_t *tkeys = reinterpret_cast<int32_t *>(tdst + SW_STAGE);
    int32_t *ckeys = tkeys + SW_STAGE;
    int32_t *tcnt = ckeys + SW_PMAX * SW_RUN;  // new rows of the tile
    int32_t *ccnt = tcnt + SW_PMAX;            // rows carried into the tile
    int32_t *fl = ccnt + SW_PMAX;              // rows written this tile (whole units)
    int32_t *wof = fl + SW_PMAX;               // first stage slot of the partition's written rows
    for (int p = tid; p < P; p += TPB) {
        run[p] = base[(size_t)blockIdx.x * P + p];
        tcnt[p] = 0;
        ccnt[p] = 0;
    }
    __syncthreads();

    auto tile = [&](const QuadT<DT> (&q)[QPT], const uint32_t (&in)[QPT]) {
        int pp[QPT][4], rk[QPT][4];
#pragma unroll
        for (int i = 0; i < QPT; ++i)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int32_t k = kq(q[i].k, u);
                pp[i][u] = -1;
                if (MR) {  // warp-aggregated: one shared atomic per distinct partition per warp (few partitions)
                    const bool ok = ((in[i] >> u) & 1u) && (uint32_t)k < (uint32_t)G;
                    const int pv = ok ? k >> gbits : -1;
                    const unsigned peers = __match_any_sync(0xffffffffu, pv);
                    const int leader = __ffs(peers) - 1;
                    int b = 0;
                    if (ok && lane == leader) b = atomicAdd(&tcnt[pv], __popc(peers));
                    b = __shfl_sync(0xffffffffu, b, leader);
                    pp[i][u] = pv;
                    rk[i][u] = b + __popc(peers & ((1u << lane) - 1u));
                } else if (((in[i] >> u) & 1u) && (uint32_t)k < (uint32_t)G) {
                    pp[i][u] = k >> gbits;
                    rk[i][u] = atomicAdd(&tcnt[pp[i][u]], 1);
                }
            }
        __syncthreads();  // B1: ranks complete
        {  // per partition (thread p): whole units written this tile, their stage offset
            const int p = tid;
            const int T = p < P ? ccnt[p] + tcnt[p] : 0;
            const int F = T & ~(SW_RUN - 1);
            int incl = F;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            int b0 = 0;
            for (int w = 0; w < warp; ++w) b0 += s_wsum[w];
            if (p < P) {
                fl[p] = F;
                wof[p] = b0 + incl - F;
            }
            if (tid == TPB - 1) s_nw = b0 + incl;
        }
        __syncthreads();  // B2
        // rows carried from the previous tile (numbers j < ccnt): staged when
        // j < F; otherwise (F == 0) they stay where they are
        for (int i = tid; i < P * SW_RUN; i += TPB) {
            const int p = i / SW_RUN, j = i % SW_RUN;
            if (j < ccnt[p] && j < fl[p]) {
                const int s_ = wof[p] + j;
                tkeys[s_] = ckeys[i];
                tvals[s_] = cvals[i];
                tdst[s_] = (DstT)(run[p] + j);
            }
        }
        __syncthreads();  // B2': the carried rows are read before new ones take their slots
#pragma unroll
        for (int i = 0; i < QPT; ++i)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int p = pp[i][u];
                if (p < 0) continue;
                const int j = ccnt[p] + rk[i][u];
                const int f = fl[p];
                if (j < f) {
                    const int s_ = wof[p] + j;
                    tkeys[s_] = kq(q[i].k, u) & (Gp - 1);
                    tvals[s_] = q[i].v(u);
                    tdst[s_] = (DstT)(run[p] + j);
                } else {
                    ckeys[p * SW_RUN + (j - f)] = kq(q[i].k, u) & (Gp - 1);
                    cvals[p * SW_RUN + (j - f)] = q[i].v(u);
                }
            }
        __syncthreads();  // B3: stage complete
        const int nw = s_nw;
        for (int s_ = tid; s_ < nw; s_ += TPB) {  // consecutive threads: consecutive rows of a run
            const DstT d = tdst[s_];
            pkeys[d] = tkeys[s_];
            pvals[d] = tvals[s_];
        }
        for (int p = tid; p < P; p += TPB) {
            const int T = ccnt[p] + tcnt[p];
            run[p] += fl[p];
            ccnt[p] = T - fl[p];
            tcnt[p] = 0;
        }
        __syncthreads();  // B4: the stage is read and the counts reset before the next tile's ranks
    };

    const int64_t nq = (row1 - row0) >> 2;
    const int64_t steps = (nq + TPB * QPT - 1) / (TPB * QPT);
    const bool vec = ((((uintptr_t)keys) | ((uintptr_t)vals)) & 15) == 0;  // (row0 is a quad multiple)
    QuadT<DT> nxt[QPT];
#pragma unroll
    for (int i = 0; i < QPT; ++i)
        if (i * TPB + tid < nq) load_quad_rt<DT>(keys, vals, row0 + 4 * (int64_t)(i * TPB + tid), nxt[i], vec);
    for (int64_t s = 0; s < steps; ++s) {
        QuadT<DT> q[QPT];
        uint32_t in[QPT];
        const int64_t q0 = s * TPB * QPT + tid;
#pragma unroll
        for (int i = 0; i < QPT; ++i) {
            q[i] = nxt[i];
            in[i] = q0 + (int64_t)i * TPB < nq ? 0xFu : 0u;
            const int64_t qn = q0 + (int64_t)(QPT + i) * TPB;
            if (qn < nq) load_quad_rt<DT>(keys, vals, row0 + 4 * qn, nxt[i], vec);
        }
        if (SW_L2PF && vec && lane == 0) {
#pragma unroll
            for (int i = 0; i < QPT; ++i) {
                const int64_t qp = (s + 2) * TPB * QPT + (int64_t)i * TPB + warp * 32;
                if (qp + 32 <= nq) {
                    l2_prefetch(keys + row0 + 4 * qp, 128 * 4);
                    l2_prefetch(vals + row0 + 4 * qp, 128 * (uint32_t)sizeof(V));
                }
            }
        }
        tile(q, in);
    }
    const int tail = (int)(row1 - row0 - 4 * nq);
    if (tail > 0) {
        QuadT<DT> q[QPT];
        uint32_t in[QPT];
#pragma unroll
        for (int i = 0; i < QPT; ++i) {
            load_partial<DT>(keys, vals, row0 + 4 * nq, (i == 0 && tid == 0) ? tail : 0, q[i]);
            in[i] = (i == 0 && tid == 0) ? (1u << tail) - 1u : 0u;
        }
        tile(q, in);
    }
    // the last, partial unit of every partition, padded
    for (int i = tid; i < P * SW_RUN; i += TPB) {
        const int p = i / SW_RUN, j = i % SW_RUN;
        if (ccnt[p] > 0) {
            const int64_t d = run[p] + j;
            pkeys[d] = j < ccnt[p] ? ckeys[i] : SW_PAD;
            pvals[d] = j < ccnt[p] ? cvals[i] : V(0);
        }
    }
}

// 6. per-partition accumulation over the work items (row ranges of one
// partition, starting on whole quads)
template <int DT, int K>
__global__ void __launch_bounds__(SW_TPB, 1)
k_sweep_acc(const int32_t *__restrict__ pkeys, const typename Fmt<DT>::V *__restrict__ pvals,
            const int64_t *__restrict__ items, const int32_t *__restrict__ bfirst, int32_t *ctrl, int32_t G,
            int gbits, int32_t *__restrict__ kglob, unsigned long long *__restrict__ slots,
            uint32_t *__restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_mm[TAB_MM];
    __shared__ int s_item;
    const int tid = threadIdx.x;
    const int Gp = 1 << gbits;
    uint32_t flags = 0;
    for (int k = 0;; ++k) {
        int it;
        if (SW_BAL) {  // this block's own items (no queue)
            it = bfirst[blockIdx.x] + k;
            if (it >= bfirst[blockIdx.x + 1]) break;
            __syncthreads();  // the previous item's table is published
        } else {
            if (tid == 0) s_item = atomicAdd(&ctrl[1], 1);
            __syncthreads();
            it = s_item;
            if (it >= ctrl[0]) break;
        }
        const int p = (int)items[3 * it];
        const int64_t r0 = items[3 * it + 1], r1 = items[3 * it + 2];
        Table<DT, K, SW_TPB, 0, false, 1> tab(smem, s_mm, min(Gp, G - p * Gp), (int64_t)p * Gp, kglob, slots);
        tab.clear();
        __syncthreads();
        const int64_t nq = (r1 - r0 + 3) >> 2;  // the last quad may hold padding rows
        constexpr int QA = 2;  // quads per thread per step (the next step's are in flight)
        const int64_t steps = (nq + SW_TPB * QA - 1) / (SW_TPB * QA);
        QuadT<DT> nxt[QA];
#pragma unroll
        for (int i = 0; i < QA; ++i)
            if (i * SW_TPB + tid < nq) load_quad<DT, true>(pkeys, pvals, r0 + 4 * (int64_t)(i * SW_TPB + tid), nxt[i]);
        // one step: the next step's quads are issued, this step's deposited
        auto step = [&](int64_t s, auto &&deposit) {
            QuadT<DT> cur[QA];
#pragma unroll
            for (int i = 0; i < QA; ++i) cur[i] = nxt[i];
            const int64_t q0 = s * SW_TPB * QA + tid;
#pragma unroll
            for (int i = 0; i < QA; ++i) {
                const int64_t qn = q0 + (int64_t)(QA + i) * SW_TPB;
                if (qn < nq) load_quad<DT, true>(pkeys, pvals, r0 + 4 * qn, nxt[i]);
            }
            if (SW_L2PF && (tid & 31) == 0) {
#pragma unroll
                for (int i = 0; i < QA; ++i) {
                    const int64_t qp = q0 + (int64_t)(2 * QA + i) * SW_TPB;  // (lane 0: the warp's first quad)
                    if (qp + 32 <= nq) {
                        l2_prefetch(pkeys + r0 + 4 * qp, 128 * 4);
                        l2_prefetch(pvals + r0 + 4 * qp, 128 * (uint32_t)sizeof(typename Fmt<DT>::V));
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < QA; ++i) {
                const QuadT<DT> &q = cur[i];
                const int64_t rq = r0 + 4 * (q0 + (int64_t)i * SW_TPB);  // first row of the quad
                uint32_t in = 0;
                if (q0 + i * SW_TPB < nq)
#pragma unroll
                    for (int u = 0; u < 4; ++u) in |= (rq + u < r1 && kq(q.k, u) >= 0) ? 1u << u : 0u;
                deposit(q, in);
            }
        };
        // (block-uniform phases, as in k_table: every mode until the table
        // streams in the uniform mode, then the uniform deposit only)
        int64_t s = 0;
        for (; s < steps && !tab.uniform(); ++s)
            step(s, [&](const QuadT<DT> &q, uint32_t in) { tab.quad(q, in, flags); });
        for (; s < steps; ++s)
            step(s, [&](const QuadT<DT> &q, uint32_t in) { tab.fast_quad(q, in, flags); });
        tab.finish();
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if ((tid & 31) == 0 && flags) atomicOr(status, flags);
}

// largest plan (partitions) that takes the replicated-read form; REPRO_SWEEP_REP_MAXP overrides (0 / 1: off)
int sweep_rep_maxp() {
    const char *e = getenv("REPRO_SWEEP_REP_MAXP");
    if (e && *e) return atoi(e);
    return SW_REP_MAXP;
}

template <int DT, int K>
int launch_sweep_t(const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws, size_t ws_bytes,
                   int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out, uint32_t *status,
                   cudaStream_t st, int *launches) {
    using V = typename Fmt<DT>::V;
    // one pass through L2 rings when the groups fit the SMs' tables
    const int rr = launch_route(DT, K, keys, vals, n, G, ws, ws_bytes, merge, acc_k, acc_C, acc_D, out, status, st,
                                launches);
    if (rr != -1) return rr;
    const SwPlan pl = sw_plan<DT, K>(n, G);
    if (pl.P > SW_PMAX) return -1;
    const bool d32 = pl.rows_cap < ((int64_t)1 << 32);  // 32-bit scatter destinations
    const size_t sm_cold = d32 ? sw_smem_cold<DT, uint32_t>() : sw_smem_cold<DT, unsigned long long>();
    const size_t sm_tab = TabGeom<DT, K, 1>::bytes(pl.Gp);  // accumulate
    const size_t sm_hot = TabGeom<DT, K, 1>::bytes(pl.Gp, TAB_HMAX);  // hot pass (+ heavy-group lane copies)
    if (sm_hot > (size_t)device_props().smem_optin - 1024) return -1;
    SwWs w = sw_carve<DT, K>(ws, n, G, pl);
    if (w.bytes > ws_bytes) return -1;
    static thread_local size_t conf_h = 0, conf_c[2][2] = {}, conf_a = 0;
    const bool mr = pl.P <= SW_MRANK;  // scatter ranks by warp match
    auto conf = [](auto kern, size_t &have, size_t want) {
        if (have >= want) return true;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want) != cudaSuccess)
            return false;
        have = want;
        return true;
    };
    // the scatter instantiation for (destination width, rank mode)
    auto with_cold = [&](auto &&fn) {
        if (d32) {
            if (mr) fn(k_sweep_cold<DT, uint32_t, true>, conf_c[0][1]);
            else fn(k_sweep_cold<DT, uint32_t, false>, conf_c[0][0]);
        } else {
            if (mr) fn(k_sweep_cold<DT, unsigned long long, true>, conf_c[1][1]);
            else fn(k_sweep_cold<DT, unsigned long long, false>, conf_c[1][0]);
        }
    };
    bool cold_ok = false;
    with_cold([&](auto kern, size_t &have) { cold_ok = conf(kern, have, sm_cold); });
    if (!conf(k_sweep_hot<DT, K>, conf_h, sm_hot) || !cold_ok || !conf(k_sweep_acc<DT, K>, conf_a, sm_tab))
        return -2;
    if (cudaMemsetAsync(ws, 0, w.zero_bytes, st) != cudaSuccess) return -2;
    int rc = 0;
    const int rep_max = sweep_rep_maxp();
    if (n > 0 && pl.P >= 2 && pl.P <= rep_max && pl.P <= pl.grid) {
        // replicated-read form: P blocks per row chunk, one partition each; no scatter
        static thread_local size_t conf_r = 0;
        if (!conf(k_sweep_hot<DT, K, true>, conf_r, sm_hot)) return -2;
        const int chunks = pl.grid / pl.P;
        int64_t chunk = (n + chunks - 1) / chunks;
        chunk = (chunk + 3) & ~(int64_t)3;
        const int grid = (int)((n + chunk - 1) / chunk) * pl.P;
        rc = traced("sweep_replicated", st, launches, [&] {
            k_sweep_hot<DT, K, true><<<grid, SW_HTPB, sm_hot, st>>>(keys, (const V *)vals, n, G, pl.gbits, chunk,
                                                                   w.bkeys, (V *)w.bvals, w.ctrl, w.hcnt, w.kglob,
                                                                   w.slots, status, pl.P);
        });
        if (rc) return rc;
    } else if (n > 0) {
        rc = traced("sweep_sample", st, launches, [&] {
            k_sw_sample<<<1, 1024, 0, st>>>(keys, n, G, pl.gbits, pl.P, w.ctrl);
        });
        if (rc) return rc;
        int64_t chunk = (n + pl.grid - 1) / pl.grid;
        chunk = (chunk + 3) & ~(int64_t)3;
        const int grid = (int)((n + chunk - 1) / chunk);
        const ColdSrc cs{w.hcnt, grid, chunk};
        rc = traced("sweep_hot", st, launches, [&] {  // returns at once when no partition is hot
            k_sweep_hot<DT, K><<<grid, SW_HTPB, sm_hot, st>>>(keys, (const V *)vals, n, G, pl.gbits, chunk, w.bkeys,
                                                             (V *)w.bvals, w.ctrl, w.hcnt, w.kglob, w.slots, status, 1);
        });
        if (rc) return rc;
        rc = traced("sweep_hist", st, launches, [&] {
            k_sw_hist<<<pl.cgrid, SW_CTPB, 0, st>>>(keys, w.bkeys, n, G, pl.gbits, pl.P, w.ctrl, cs, w.cnt, status);
        });
        if (rc) return rc;
        rc = traced("sweep_scan", st, launches, [&] {
            k_sw_scan<<<1, 1024, 0, st>>>(w.cnt, pl.cgrid, pl.P, w.pstart, w.pkeys, w.items, w.bfirst, pl.grid,
                                          w.ctrl);
        });
        if (rc) return rc;
        rc = traced("sweep_scatter", st, launches, [&] {
            with_cold([&](auto kern, size_t &) {
                kern<<<pl.cgrid, SW_STPB, sm_cold, st>>>(keys, (const V *)vals, n, w.bkeys, (const V *)w.bvals, G,
                                                         pl.gbits, pl.P, w.cnt, w.pkeys, (V *)w.pvals, w.ctrl, cs);
            });
        });
        if (rc) return rc;
        rc = traced("sweep_accumulate", st, launches, [&] {
            k_sweep_acc<DT, K><<<device_props().sms, SW_TPB, sm_tab, st>>>(
                w.pkeys, (const V *)w.pvals, w.items, w.bfirst, w.ctrl, G, pl.gbits, w.kglob, w.slots, status);
        });
        if (rc) return rc;
    }
    if (!out && !acc_k) return 0;  // deposit only (the split form: the caller reads the slot table)
    return launch_fold(DT, K, G, w.kglob, w.slots, merge, acc_k, acc_C, acc_D, out, status, st, launches);
}

}  // namespace

int sweep_max_groups(int K, int DT) {
#define SWG(dt, k) \
    if (DT == dt && K == k) return SW_PMAX << sw_gbits<dt, k>();
    SWG(1, 1) SWG(1, 2) SWG(1, 3) SWG(1, 4) SWG(0, 1) SWG(0, 2) SWG(0, 3) SWG(0, 4)
#undef SWG
    return 0;
}

size_t sweep_workspace_bytes(int64_t n, int32_t G, int K, int DT) {
#define SWB(dt, k)                                          \
    if (DT == dt && K == k) {                               \
        const SwPlan pl = sw_plan<dt, k>(n, G);             \
        return std::max(sw_carve<dt, k>(nullptr, n, G, pl).bytes,                                   \
                        route_mode() ? route_workspace_bytes(G, k, dt) : (size_t)0); /* (rings: opt-in) */ \
    }
    SWB(1, 1) SWB(1, 2) SWB(1, 3) SWB(1, 4) SWB(0, 1) SWB(0, 2) SWB(0, 3) SWB(0, 4)
#undef SWB
    return 0;
}

int launch_sweep(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws,
                 size_t ws_bytes, int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out,
                 uint32_t *status, cudaStream_t st, int *launches) {
#define SWL(dt, k)          \
    if (DT == dt && K == k) \
        return launch_sweep_t<dt, k>(keys, vals, n, G, ws, ws_bytes, merge, acc_k, acc_C, acc_D, out, status, st, launches);
    SWL(1, 1) SWL(1, 2) SWL(1, 3) SWL(1, 4) SWL(0, 1) SWL(0, 2) SWL(0, 3) SWL(0, 4)
#undef SWL
    return -1;
}

}  // namespace repro
