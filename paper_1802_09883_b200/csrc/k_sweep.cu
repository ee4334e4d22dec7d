// k_sweep.cu -- the high-cardinality GroupBy:
// PartitionAndAggregate (Alg. 4) in two passes over the
// rows, for group counts above the on-chip table's capacity.
//
// Groups are split into P <= 256 partitions of Gp = 2^gbits consecutive keys
// (Gp sized so one partition's table fits on chip, F = f^d with d = 1,
// PAPER.md:1054-1058).
//   1. k_sw_sample   reads 8192 evenly spaced keys; a partition holding >= 1/8
//                    of them is HOT (skew, e.g. Zipf's head).
//   2. k_sweep       one pass over the rows, one persistent block per SM over
//                    a contiguous row range: hot-partition rows are deposited
//                    on chip right away (table_core.cuh, the heavy partition
//                    never goes back to HBM); every other row is ranked within
//                    its tile per partition, staged in shared memory in
//                    partition order, and written out in whole UNITS (8 fp64 /
//                    16 fp32 rows: full 32-byte sectors of keys and values)
//                    into the block's current CHUNK of that partition (chunks
//                    come from a global pool, one atomic per chunk).  Rows
//                    short of a unit wait in shared memory for the next tile.
//   3. k_sw_lists    chunk lists per partition and work items (<= CPI chunks).
//   4. k_sweep_acc   persistent blocks pull work items and run the on-chip
//                    table over the item's chunks (local keys).
// Both tables publish into the absolute-level slot table (kglob, slots), which
// k_fold (k_state.cu) turns into canonical states and Eq. 1 read-outs.  Each
// group lives in exactly one partition; the order of rows inside a partition
// is irrelevant (the accumulator is associative).
//
// HBM traffic: the rows are read once; cold rows are written once and read
// once more (12 B per binary64 row each way); hot rows are read once.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"
#include "table_core.cuh"

#include <algorithm>

namespace repro {

namespace {

constexpr int SW_TPB = 512;
constexpr int SW_NW = SW_TPB / 32;
constexpr int SW_TILE = 4 * SW_TPB;    // rows per sweep tile (one quad per thread)
constexpr int SW_PMAX = 256;           // partitions of one sweep
constexpr int SW_CHR = SW_TILE + 256;  // rows per chunk (>= TILE + unit: a tile's units span <= 2 chunks)
constexpr int SW_SAMPLE = 8192;
constexpr int SW_CPI = 256;            // chunks per accumulate work item
constexpr int SW_TABLE_MAX = 168 * 1024;
// control words: [0] chunks allocated, [1] work items, [2] queue head, [3] hot partition
constexpr int SW_CTRL = 8;

template <int DT>
constexpr int sw_unit() { return DT == 1 ? 8 : 16; }

template <int DT, int K>
int sw_gbits() {  // largest power-of-two partition whose table fits SW_TABLE_MAX
    int b = 13;
    while (b > 8 && TabGeom<DT, K>::bytes(1 << b) > SW_TABLE_MAX) --b;
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
    int gbits, Gp, P, grid;
    int64_t max_chunks, max_items;
};

template <int DT, int K>
SwPlan sw_plan(int64_t n, int32_t G) {
    SwPlan pl{};
    pl.gbits = sw_gbits<DT, K>();
    pl.Gp = 1 << pl.gbits;
    pl.P = (int)(((int64_t)G + pl.Gp - 1) >> pl.gbits);
    pl.grid = device_props().sms;
    pl.max_chunks = (n + SW_CHR - 1) / SW_CHR + (int64_t)pl.grid * pl.P + 1;
    pl.max_items = pl.P + pl.max_chunks / SW_CPI + 1;
    return pl;
}

template <int DT, int K>
size_t sw_smem(const SwPlan &pl) {
    using V = typename Fmt<DT>::V;
    constexpr int U = sw_unit<DT>();
    size_t b = (TabGeom<DT, K>::bytes(pl.Gp) + 15) & ~(size_t)15;
    b += (size_t)SW_TILE * (4 + sizeof(V));
    b += (size_t)pl.P * U * (4 + sizeof(V));
    b += (size_t)pl.P * (9 * 4 + 2 * 8);
    return b;
}

struct SwWs {
    int32_t *kglob;
    unsigned long long *slots;
    int32_t *ctrl;
    size_t zero_bytes;  // kglob .. ctrl (one memset)
    int32_t *ckeys;
    void *cvals;
    int32_t *chunk_part, *chunk_rows, *plist, *items;
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
    w.zero_bytes = o;
    w.ckeys = (int32_t *)take(4 * (size_t)pl.max_chunks * SW_CHR);
    w.cvals = take(sizeof(V) * (size_t)pl.max_chunks * SW_CHR);
    w.chunk_part = (int32_t *)take(4 * (size_t)pl.max_chunks);
    w.chunk_rows = (int32_t *)take(4 * (size_t)pl.max_chunks);
    w.plist = (int32_t *)take(4 * (size_t)pl.max_chunks);
    w.items = (int32_t *)take(12 * (size_t)pl.max_items);
    w.bytes = o;
    return w;
}

// 1. hot partition from evenly spaced keys (performance only: any choice
// gives the same bits)
__global__ void __launch_bounds__(1024) k_sw_sample(const int32_t *__restrict__ keys, int64_t n, int32_t G, int gbits,
                                                    int P, int32_t *ctrl) {
    __shared__ int cnt[SW_PMAX];
    __shared__ unsigned long long best;
    const int tid = threadIdx.x;
    for (int i = tid; i < SW_PMAX; i += 1024) cnt[i] = 0;
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
    if (tid == 0) {
        const int c = (int)(best >> 32);
        const int samples = (int)min((int64_t)SW_SAMPLE, n);
        ctrl[3] = (c > 0 && 8 * c >= samples) ? SW_PMAX - 1 - (int)(best & 0xFFFFFFFFu) : -1;
    }
}

// 2. the sweep
template <int DT, int K>
__global__ void __launch_bounds__(SW_TPB, 1)
k_sweep(const int32_t *__restrict__ keys, const typename Fmt<DT>::V *__restrict__ vals, int64_t n, int32_t G,
        int gbits, int P, int64_t chunk, int32_t *__restrict__ ckeys, typename Fmt<DT>::V *__restrict__ cvals,
        int32_t *__restrict__ chunk_part, int32_t *__restrict__ chunk_rows, int64_t max_chunks,
        int32_t *__restrict__ ctrl, int32_t *__restrict__ kglob, unsigned long long *__restrict__ slots,
        uint32_t *__restrict__ status) {
    using V = typename Fmt<DT>::V;
    constexpr int U = sw_unit<DT>();
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_mm[TAB_MM];
    __shared__ int s_wsum[SW_NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Gp = 1 << gbits;
    const int hot = ctrl[3];
    const int64_t row0 = (int64_t)blockIdx.x * chunk;
    const int64_t row1 = min(n, row0 + chunk);
    if (row0 >= row1) return;

    // shared memory: hot table | tile stage | leftover stage | per-partition words
    const size_t tb = (TabGeom<DT, K>::bytes(Gp) + 15) & ~(size_t)15;
    int32_t *tkeys = reinterpret_cast<int32_t *>(smem + tb);
    V *tvals = reinterpret_cast<V *>(tkeys + SW_TILE);
    int32_t *lkeys = reinterpret_cast<int32_t *>(tvals + SW_TILE);
    V *lvals = reinterpret_cast<V *>(lkeys + P * U);
    int64_t *dst0 = reinterpret_cast<int64_t *>(lvals + P * U);
    int64_t *dst1 = dst0 + P;
    int32_t *tcnt = reinterpret_cast<int32_t *>(dst1 + P);
    int32_t *left = tcnt + P;   // rows waiting in the leftover stage
    int32_t *off = left + P;    // tile-stage offset of this tile's rows
    int32_t *lcur = off + P;    // leftovers at the start of this tile
    int32_t *tcur = lcur + P;   // this tile's rows
    int32_t *full = tcur + P;   // whole units flushed this tile
    int32_t *msplit = full + P; // units that go to the current chunk
    int32_t *cur = msplit + P;  // the block's current chunk of each partition (-1: none)
    int32_t *fill = cur + P;    // rows used in it

    const int Gh = hot >= 0 ? min(Gp, G - hot * Gp) : 1;
    Table<DT, K, SW_TPB> tab(smem, s_mm, Gh, hot >= 0 ? (int64_t)hot * Gp : 0, kglob, slots);
    if (hot >= 0) tab.clear();
    for (int p = tid; p < P; p += SW_TPB) {
        tcnt[p] = 0;
        left[p] = 0;
        cur[p] = -1;
        fill[p] = 0;
    }
    uint32_t flags = 0;
    __syncthreads();

    auto alloc = [&](int p) -> int {
        const int c = atomicAdd(&ctrl[0], 1);
        if (c >= max_chunks) { flags |= FLAG_EINVAL; return -1; }  // sizing guarantees this never happens
        chunk_part[c] = p;
        return c;
    };

    // one tile: the quad of this thread (`in` bit u: row u exists)
    auto tile = [&](const QuadT<DT> &q, uint32_t in) {
        int pp[4], rk[4], lk[4];
        uint32_t hin = 0;
        QuadT<DT> hq = q;
        int hk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t k = kq(q.k, u);
            pp[u] = -1;
            hk[u] = 0;
            if (!((in >> u) & 1u)) continue;
            if ((uint32_t)k >= (uint32_t)G) { flags |= FLAG_EKEY; continue; }
            const int p = k >> gbits;
            lk[u] = k & (Gp - 1);
            if (p == hot) {
                hin |= 1u << u;
                hk[u] = lk[u];
            } else {
                pp[u] = p;
                rk[u] = atomicAdd(&tcnt[p], 1);
            }
        }
        if (hot >= 0) {  // block-uniform
            hq.k = make_int4(hk[0], hk[1], hk[2], hk[3]);
            tab.quad(hq, hin, flags);
        }
        __syncthreads();  // B1: ranks complete
        // per partition: tile-stage offsets (block scan), units to flush,
        // destination chunks
        {
            const int p = tid;
            const int T = p < P ? tcnt[p] : 0;
            int incl = T;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            int base = 0;
            for (int w = 0; w < warp; ++w) base += s_wsum[w];
            if (p < P) {
                tcnt[p] = 0;
                off[p] = base + incl - T;
                const int L = left[p], tot = L + T, f = tot / U;
                lcur[p] = L;
                tcur[p] = T;
                full[p] = f;
                left[p] = tot - f * U;
                if (f > 0) {
                    int c = cur[p], fl = fill[p];
                    if (c < 0) { c = alloc(p); fl = 0; }
                    const int m = min(f, (SW_CHR - fl) / U);
                    dst0[p] = c < 0 ? -1 : (int64_t)c * SW_CHR + fl;
                    fl += m * U;
                    if (m < f) {
                        if (c >= 0) chunk_rows[c] = fl;
                        c = alloc(p);
                        fl = (f - m) * U;
                        dst1[p] = c < 0 ? -1 : (int64_t)c * SW_CHR;
                    }
                    msplit[p] = m;
                    cur[p] = c;
                    fill[p] = fl;
                }
            }
        }
        __syncthreads();  // B2
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (pp[u] < 0) continue;
            const int s = off[pp[u]] + rk[u];
            tkeys[s] = lk[u];
            tvals[s] = q.v(u);
        }
        __syncthreads();  // B3: tile stage complete
        // flush: one warp per partition, 32 / U units per warp instruction
        for (int p = warp; p < P; p += SW_NW) {
            const int f = full[p], L = lcur[p], tot = L + tcur[p], o = off[p];
            if (f > 0) {
                const int m = msplit[p];
                const int64_t d0 = dst0[p], d1 = dst1[p];
                for (int j0 = 0; j0 < f; j0 += 32 / U) {
                    const int j = j0 + lane / U, t = lane % U;
                    if (j < f) {
                        const int s = j * U + t;
                        const int32_t kk = s < L ? lkeys[p * U + s] : tkeys[o + s - L];
                        const V vv = s < L ? lvals[p * U + s] : tvals[o + s - L];
                        const int64_t d = j < m ? d0 + (int64_t)j * U : d1 + (int64_t)(j - m) * U;
                        if (d >= 0) {
                            ckeys[d + t] = kk;
                            cvals[d + t] = vv;
                        }
                    }
                }
                __syncwarp();
            }
            // rows short of a unit wait in the leftover stage
            for (int s = max(L, f * U) + lane; s < tot; s += 32) {
                lkeys[p * U + s - f * U] = tkeys[o + s - L];
                lvals[p * U + s - f * U] = tvals[o + s - L];
            }
        }
        // (the next tile's rank atomics touch only tcnt; its stage writes
        // come after its B2)
    };

    const int64_t nq = (row1 - row0) >> 2;
    const int64_t steps = (nq + SW_TPB - 1) / SW_TPB;
    QuadT<DT> nxt;
    if (tid < nq) load_quad<DT, true>(keys, vals, row0 + 4 * (int64_t)tid, nxt);
    for (int64_t s = 0; s < steps; ++s) {
        const QuadT<DT> q = nxt;
        const int64_t qi = s * SW_TPB + tid;
        if (qi + SW_TPB < nq) load_quad<DT, true>(keys, vals, row0 + 4 * (qi + SW_TPB), nxt);
        tile(q, qi < nq ? 0xFu : 0u);
    }
    const int tail = (int)(row1 - row0 - 4 * nq);
    if (tail > 0) {
        QuadT<DT> t;
        load_partial<DT>(keys, vals, row0 + 4 * nq, tid == 0 ? tail : 0, t);
        tile(t, tid == 0 ? (1u << tail) - 1u : 0u);
    }
    __syncthreads();
    // the last rows of every partition: one partial unit, padded to whole quads
    for (int p = tid; p < P; p += SW_TPB) {
        const int nl = left[p];
        int c = cur[p], fl = fill[p];
        if (nl > 0) {
            const int padded = (nl + 3) & ~3;
            if (c < 0 || fl + padded > SW_CHR) {
                if (c >= 0) chunk_rows[c] = fl;
                c = alloc(p);
                fl = 0;
            }
            if (c >= 0) {
                const int64_t d = (int64_t)c * SW_CHR + fl;
                for (int i = 0; i < padded; ++i) {
                    ckeys[d + i] = i < nl ? lkeys[p * U + i] : -1;
                    cvals[d + i] = i < nl ? lvals[p * U + i] : V(0);
                }
                fl += padded;
            }
        }
        if (c >= 0) chunk_rows[c] = fl;
    }
    if (hot >= 0) tab.finish();
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0 && flags) atomicOr(status, flags);
}

// 3. chunk lists per partition and work items (single block)
__global__ void __launch_bounds__(1024) k_sw_lists(const int32_t *__restrict__ chunk_part, int P,
                                                   int32_t *__restrict__ plist, int32_t *__restrict__ items,
                                                   int32_t *ctrl) {
    __shared__ int pc[SW_PMAX], ps[SW_PMAX + 1], pi[SW_PMAX + 1], cursor[SW_PMAX];
    const int tid = threadIdx.x;
    const int nch = ctrl[0];
    for (int p = tid; p < SW_PMAX; p += 1024) { pc[p] = 0; cursor[p] = 0; }
    __syncthreads();
    for (int c = tid; c < nch; c += 1024) atomicAdd(&pc[chunk_part[c]], 1);
    __syncthreads();
    if (tid == 0) {
        int a = 0, b = 0;
        for (int p = 0; p < P; ++p) {
            ps[p] = a;
            pi[p] = b;
            a += pc[p];
            b += (pc[p] + SW_CPI - 1) / SW_CPI;
        }
        ps[P] = a;
        pi[P] = b;
        ctrl[1] = b;
        ctrl[2] = 0;
    }
    __syncthreads();
    for (int c = tid; c < nch; c += 1024) {
        const int p = chunk_part[c];
        plist[ps[p] + atomicAdd(&cursor[p], 1)] = c;
    }
    for (int p = tid; p < P; p += 1024)
        for (int i = pi[p], c0 = ps[p]; i < pi[p + 1]; ++i, c0 += SW_CPI) {
            items[3 * i] = p;
            items[3 * i + 1] = c0;
            items[3 * i + 2] = min(c0 + SW_CPI, ps[p + 1]);
        }
}

// 4. per-partition accumulation over the chunks of each work item
template <int DT, int K>
__global__ void __launch_bounds__(SW_TPB, 1)
k_sweep_acc(const int32_t *__restrict__ ckeys, const typename Fmt<DT>::V *__restrict__ cvals,
            const int32_t *__restrict__ plist, const int32_t *__restrict__ chunk_rows,
            const int32_t *__restrict__ items, int32_t *ctrl, int32_t G, int gbits, int32_t *__restrict__ kglob,
            unsigned long long *__restrict__ slots, uint32_t *__restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_mm[TAB_MM];
    __shared__ int s_item;
    __shared__ int s_cid[SW_CPI], s_pre[SW_CPI + 1];
    const int tid = threadIdx.x;
    const int Gp = 1 << gbits;
    uint32_t flags = 0;
    for (;;) {
        if (tid == 0) s_item = atomicAdd(&ctrl[2], 1);
        __syncthreads();
        const int it = s_item;
        if (it >= ctrl[1]) break;
        const int p = items[3 * it], c0 = items[3 * it + 1], nc = items[3 * it + 2] - c0;
        Table<DT, K, SW_TPB> tab(smem, s_mm, min(Gp, G - p * Gp), (int64_t)p * Gp, kglob, slots);
        tab.clear();
        if (tid < nc) s_cid[tid] = plist[c0 + tid];
        __syncthreads();
        if (tid == 0) {  // quad prefix over the item's chunks
            int a = 0;
            for (int i = 0; i < nc; ++i) {
                s_pre[i] = a;
                a += chunk_rows[s_cid[i]] >> 2;
            }
            s_pre[nc] = a;
        }
        __syncthreads();
        const int nq = s_pre[nc];
        auto row_of = [&](int qi) -> int64_t {  // first row of quad qi in the chunk storage
            int lo = 0, hi = nc - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_pre[mid] <= qi) lo = mid;
                else hi = mid - 1;
            }
            return (int64_t)s_cid[lo] * SW_CHR + 4 * (int64_t)(qi - s_pre[lo]);
        };
        const int steps = (nq + SW_TPB - 1) / SW_TPB;
        QuadT<DT> nxt;
        if (tid < nq) load_quad<DT, true>(ckeys, cvals, row_of(tid), nxt);
        for (int s = 0; s < steps; ++s) {
            const QuadT<DT> q = nxt;
            const int qi = s * SW_TPB + tid;
            if (qi + SW_TPB < nq) load_quad<DT, true>(ckeys, cvals, row_of(qi + SW_TPB), nxt);
            uint32_t in = 0;
            if (qi < nq) in = (q.k.x >= 0 ? 1u : 0u) | (q.k.y >= 0 ? 2u : 0u) | (q.k.z >= 0 ? 4u : 0u) |
                              (q.k.w >= 0 ? 8u : 0u);
            tab.quad(q, in, flags);
        }
        tab.finish();
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if ((tid & 31) == 0 && flags) atomicOr(status, flags);
}

template <int DT, int K>
int launch_sweep_t(const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws, size_t ws_bytes,
                   int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out, uint32_t *status,
                   cudaStream_t st, int *launches) {
    using V = typename Fmt<DT>::V;
    const SwPlan pl = sw_plan<DT, K>(n, G);
    if (pl.P > SW_PMAX) return -1;
    const size_t sm_sweep = sw_smem<DT, K>(pl);
    const size_t sm_acc = TabGeom<DT, K>::bytes(pl.Gp);
    if (sm_sweep > (size_t)device_props().smem_optin - 1024) return -1;
    SwWs w = sw_carve<DT, K>(ws, n, G, pl);
    if (w.bytes > ws_bytes) return -1;
    static thread_local size_t conf_s = 0, conf_a = 0;
    if (conf_s < sm_sweep) {
        if (cudaFuncSetAttribute(k_sweep<DT, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sweep) !=
            cudaSuccess)
            return -2;
        conf_s = sm_sweep;
    }
    if (conf_a < sm_acc) {
        if (cudaFuncSetAttribute(k_sweep_acc<DT, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_acc) !=
            cudaSuccess)
            return -2;
        conf_a = sm_acc;
    }
    if (cudaMemsetAsync(ws, 0, w.zero_bytes, st) != cudaSuccess) return -2;
    int rc = 0;
    if (n > 0) {
        rc = traced("sweep_sample", st, launches, [&] {
            k_sw_sample<<<1, 1024, 0, st>>>(keys, n, G, pl.gbits, pl.P, w.ctrl);
        });
        if (rc) return rc;
        int64_t chunk = (n + pl.grid - 1) / pl.grid;
        chunk = (chunk + 3) & ~(int64_t)3;
        const int grid = (int)((n + chunk - 1) / chunk);
        rc = traced("sweep", st, launches, [&] {
            k_sweep<DT, K><<<grid, SW_TPB, sm_sweep, st>>>(keys, (const V *)vals, n, G, pl.gbits, pl.P, chunk,
                                                          w.ckeys, (V *)w.cvals, w.chunk_part, w.chunk_rows,
                                                          pl.max_chunks, w.ctrl, w.kglob, w.slots, status);
        });
        if (rc) return rc;
        rc = traced("sweep_lists", st, launches, [&] {
            k_sw_lists<<<1, 1024, 0, st>>>(w.chunk_part, pl.P, w.plist, w.items, w.ctrl);
        });
        if (rc) return rc;
        rc = traced("sweep_accumulate", st, launches, [&] {
            k_sweep_acc<DT, K><<<device_props().sms, SW_TPB, sm_acc, st>>>(
                w.ckeys, (const V *)w.cvals, w.plist, w.chunk_rows, w.items, w.ctrl, G, pl.gbits, w.kglob, w.slots,
                status);
        });
        if (rc) return rc;
    }
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
        return sw_carve<dt, k>(nullptr, n, G, pl).bytes;    \
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
