// k_partition.cu -- high-cardinality path:
// PartitionAndAggregate (Alg. 4) on the GPU.
//
//   1. k_part_hist     per-block histogram of partition ids p = key >> s
//                      (contiguous key ranges of Gp = 2^s groups), EKEY check
//   2. k_part_colscan  per partition: offsets of every block inside it
//   3. k_part_plan     exclusive scan of partition sizes; split every
//                      partition into work items of <= CH rows (so skewed
//                      partitions are shared by many blocks)
//   4. k_part_scatter  rows -> partition order (ParallelPartition, PAPER.md:
//                      1054-1065; the order inside a partition is irrelevant
//                      because the accumulator is associative)
//   5. k_part_accumulate persistent blocks pull work items and run the
//                      on-chip table code (onchip_core.cuh) on Gp local groups,
//                      writing one partial state per (item, group)
//   6. k_part_merge    per group: max of the items' window tops, realign, add
//                      (the shared-table merge of Alg. 4 lines 6-9 via
//                      operator+=(repro)), canonicalise,
//                      Eq. 1 read-out / merge into an accumulator.
// Each group lives in exactly one partition, so no group is merged across
// partitions.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"

#include <algorithm>

namespace repro {

namespace {

constexpr int PART_LOG_GP = 10;               // Gp = 1024 groups per partition
constexpr int PART_GP = 1 << PART_LOG_GP;
constexpr int64_t PART_CH = 1 << 14;          // minimum rows per work item
constexpr int HIST_TPB = 512;
constexpr size_t PALIGN = 256;

inline size_t al(size_t x) { return (x + PALIGN - 1) / PALIGN * PALIGN; }

struct Plan {
    int64_t ch;     // rows per work item
    int P;          // partitions
    int B;          // histogram / scatter blocks
    int64_t chunk;  // rows per histogram block
    int64_t max_items;
};

Plan make_plan(int64_t n, int32_t G) {
    Plan pl;
    pl.P = (int)(((int64_t)G + PART_GP - 1) >> PART_LOG_GP);
    pl.B = std::max(1, std::min<int>(2 * device_props().sms, (int)((n + 65535) / 65536)));
    pl.chunk = (n + pl.B - 1) / pl.B;
    pl.chunk = (pl.chunk + 3) / 4 * 4;
    if (pl.chunk == 0) pl.chunk = 4;
    pl.B = (int)std::max<int64_t>(1, (n + pl.chunk - 1) / pl.chunk);
    // work items: ~8 per SM over the whole input, at least PART_CH rows
    pl.ch = std::max<int64_t>(PART_CH, (n + 8 * device_props().sms - 1) / (8 * device_props().sms));
    pl.max_items = (n + pl.ch - 1) / pl.ch + pl.P;
    return pl;
}

struct PartWs {
    int32_t *pkeys;
    void *pvals;
    uint32_t *hist;   // [B][P]
    int64_t *ptot;    // [P]    partition sizes
    int64_t *base;    // [P+1]  first row of each partition
    int64_t *pitem;   // [P+1]  first work item of each partition
    int64_t *items;   // [max_items][2] row range
    int32_t *iown;    // [max_items] partition of each item
    int32_t *ctrl;    // [0] number of items, [1] work-queue head
    int32_t *pk;      // [max_items][Gp]
    int64_t *pT;      // [max_items][Gp][K]
    size_t bytes;
};

PartWs carve(void *ws, int64_t n, int32_t G, int K, int DT, const Plan &pl) {
    PartWs w{};
    char *b = (char *)ws;
    size_t o = 0;
    const size_t vsz = DT == 1 ? 8 : 4;
    auto take = [&](size_t bytes) { char *p = b + o; o += al(bytes); return p; };
    w.pkeys = (int32_t *)take(4 * (size_t)n + 16);
    w.pvals = take(vsz * (size_t)n + 16);
    w.hist = (uint32_t *)take(4 * (size_t)pl.B * pl.P);
    w.ptot = (int64_t *)take(8 * (size_t)pl.P);
    w.base = (int64_t *)take(8 * ((size_t)pl.P + 1));
    w.pitem = (int64_t *)take(8 * ((size_t)pl.P + 1));
    w.items = (int64_t *)take(16 * (size_t)pl.max_items);
    w.iown = (int32_t *)take(4 * (size_t)pl.max_items);
    w.ctrl = (int32_t *)take(16);
    w.pk = (int32_t *)take(4 * (size_t)pl.max_items * PART_GP);
    w.pT = (int64_t *)take(8 * (size_t)pl.max_items * PART_GP * K);
    w.bytes = o;
    return w;
}

__global__ void __launch_bounds__(HIST_TPB)
k_part_hist(const int32_t *__restrict__ keys, int64_t n, int32_t G, int P, int64_t chunk, uint32_t *hist,
            uint32_t *status) {
    extern __shared__ uint32_t bins[];
    for (int p = threadIdx.x; p < P; p += HIST_TPB) bins[p] = 0;
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(n, r0 + chunk);  // r0 % 4 == 0
    uint32_t bad = 0;
    const int64_t v1 = r0 + ((r1 - r0) & ~(int64_t)3);
    for (int64_t r = r0 + 4 * (int64_t)threadIdx.x; r < v1; r += 4 * HIST_TPB) {
        const int4 k4 = __ldg(reinterpret_cast<const int4 *>(keys + r));
        const int kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if ((uint32_t)kk[j] < (uint32_t)G) atomicAdd(&bins[kk[j] >> PART_LOG_GP], 1u);
            else bad = FLAG_EKEY;
        }
    }
    for (int64_t r = v1 + threadIdx.x; r < r1; r += HIST_TPB) {
        const int k = __ldg(keys + r);
        if ((uint32_t)k < (uint32_t)G) atomicAdd(&bins[k >> PART_LOG_GP], 1u);
        else bad = FLAG_EKEY;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += HIST_TPB) hist[(size_t)blockIdx.x * P + p] = bins[p];
    bad = __reduce_or_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(status, bad);
}

// per partition p: hist[b][p] <- rows of p in blocks < b; ptot[p] <- total
__global__ void k_part_colscan(uint32_t *hist, int B, int P, int64_t *ptot) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    int64_t run = 0;
    for (int b = 0; b < B; ++b) {
        const uint32_t c = hist[(size_t)b * P + p];
        hist[(size_t)b * P + p] = (uint32_t)run;
        run += c;
    }
    ptot[p] = run;
}

// single block: base[] = exclusive scan of ptot, pitem[] = exclusive scan of
// the items per partition, then the item table
__global__ void __launch_bounds__(1024) k_part_plan(const int64_t *ptot, int P, int64_t chunk_rows, int64_t *base,
                                                    int64_t *pitem, int64_t *items, int32_t *iown, int32_t *ctrl) {
    __shared__ int64_t wsum[2][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (P + 1023) / 1024;
    const int p0 = min(tid * per, P), p1 = min(p0 + per, P);
    int64_t rows = 0, its = 0;
    for (int p = p0; p < p1; ++p) {
        rows += ptot[p];
        its += (ptot[p] + chunk_rows - 1) / chunk_rows;
    }
    int64_t ir = rows, ii = its;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t a = __shfl_up_sync(0xffffffffu, ir, o), b = __shfl_up_sync(0xffffffffu, ii, o);
        if (lane >= o) { ir += a; ii += b; }
    }
    if (lane == 31) { wsum[0][warp] = ir; wsum[1][warp] = ii; }
    __syncthreads();
    int64_t pr = ir - rows, pi = ii - its;
    for (int w = 0; w < warp; ++w) { pr += wsum[0][w]; pi += wsum[1][w]; }
    for (int p = p0; p < p1; ++p) {
        base[p] = pr;
        pitem[p] = pi;
        const int64_t c = (ptot[p] + chunk_rows - 1) / chunk_rows;
        for (int64_t i = 0; i < c; ++i) {
            items[2 * (pi + i)] = pr + i * chunk_rows;
            items[2 * (pi + i) + 1] = min(pr + (i + 1) * chunk_rows, pr + ptot[p]);
            iown[pi + i] = p;
        }
        pr += ptot[p];
        pi += c;
    }
    if (tid == 1023) {
        base[P] = pr;
        pitem[P] = pi;
        ctrl[0] = (int32_t)pi;
        ctrl[1] = 0;
    }
}

// Direct scatter (one 32-bit shared cursor per partition): best when there
// are very few partitions (runs are long anyway) or too many to stage.
template <typename V>
__global__ void __launch_bounds__(HIST_TPB)
k_part_scatter_direct(const int32_t *__restrict__ keys, const V *__restrict__ vals, int64_t n, int32_t G, int P,
                      int64_t chunk, const uint32_t *hist, const int64_t *base, int32_t *pkeys, V *pvals) {
    extern __shared__ uint32_t cursor_d[];
    for (int p = threadIdx.x; p < P; p += HIST_TPB)
        cursor_d[p] = (uint32_t)(base[p] + hist[(size_t)blockIdx.x * P + p]);
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(n, r0 + chunk);  // r0 % 4 == 0
    const int64_t v1 = r0 + ((r1 - r0) & ~(int64_t)3);
    for (int64_t r = r0 + 4 * (int64_t)threadIdx.x; r < v1; r += 4 * HIST_TPB) {
        const int4 k4 = __ldg(reinterpret_cast<const int4 *>(keys + r));
        const int kk[4] = {k4.x, k4.y, k4.z, k4.w};
        V vv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) vv[j] = __ldg(vals + r + j);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if ((uint32_t)kk[j] >= (uint32_t)G) continue;
            const uint32_t pos = atomicAdd(&cursor_d[kk[j] >> PART_LOG_GP], 1u);
            pkeys[pos] = kk[j] & (PART_GP - 1);
            pvals[pos] = vv[j];
        }
    }
    for (int64_t r = v1 + threadIdx.x; r < r1; r += HIST_TPB) {
        const int k = __ldg(keys + r);
        if ((uint32_t)k >= (uint32_t)G) continue;
        const uint32_t pos = atomicAdd(&cursor_d[k >> PART_LOG_GP], 1u);
        pkeys[pos] = k & (PART_GP - 1);
        pvals[pos] = __ldg(vals + r);
    }
}

// Scatter with tile-local sorting: each tile of SC_TILE rows is first grouped
// by partition in shared memory (rank from a shared histogram, offsets from a
// block scan), then written out so that consecutive threads store consecutive
// rows of the same partition (coalesced runs instead of one line per lane).
constexpr int SC_TPB = 512;
constexpr int SC_R = 8;
constexpr int SC_TILE = SC_TPB * SC_R;

template <typename V>
struct ScatterSmem {
    // [P] per-partition: next global row of this block, tile count, tile start
    static size_t bytes(int P) { return (size_t)12 * P + 64 * 4 + (size_t)SC_TILE * (sizeof(V) + 4 + 2) + 64; }
};

template <typename V>
__global__ void __launch_bounds__(SC_TPB)
k_part_scatter(const int32_t *__restrict__ keys, const V *__restrict__ vals, int64_t n, int32_t G, int P,
               int64_t chunk, const uint32_t *hist, const int64_t *base, int32_t *pkeys, V *pvals) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint32_t *cursor = reinterpret_cast<uint32_t *>(sm);  // [P] global row (n < 2^32)
    uint32_t *tcnt = cursor + P;                           // [P] rows of the tile per partition
    uint32_t *tstart = tcnt + P;                           // [P] tile-local start
    uint32_t *wsum = tstart + P;                           // [32] scan scratch
    V *sval = reinterpret_cast<V *>(sm + (((size_t)12 * P + 64 * 4 + 15) & ~(size_t)15));
    int32_t *skey = reinterpret_cast<int32_t *>(sval + SC_TILE);
    uint16_t *spart = reinterpret_cast<uint16_t *>(skey + SC_TILE);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int p = tid; p < P; p += SC_TPB) {
        cursor[p] = (uint32_t)(base[p] + hist[(size_t)blockIdx.x * P + p]);
        tcnt[p] = 0;
    }
    __syncthreads();
    const int cper = (P + SC_TPB - 1) / SC_TPB;
    const int s0 = min(tid * cper, P), s1 = min(s0 + cper, P);
    const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(n, r0 + chunk);
    for (int64_t tb = r0; tb < r1; tb += SC_TILE) {
        int kk[SC_R], pp[SC_R];
        uint32_t rk[SC_R];
        V vv[SC_R];
#pragma unroll
        for (int i = 0; i < SC_R; ++i) {
            const int64_t r = tb + (int64_t)i * SC_TPB + tid;
            kk[i] = -1;
            if (r < r1) {
                kk[i] = __ldg(keys + r);
                vv[i] = __ldg(vals + r);
            }
            pp[i] = (uint32_t)kk[i] < (uint32_t)G ? (kk[i] >> PART_LOG_GP) : -1;
            rk[i] = pp[i] >= 0 ? atomicAdd(&tcnt[pp[i]], 1u) : 0u;
        }
        __syncthreads();
        // exclusive scan of the tile counts over the partitions
        uint32_t local = 0;
        for (int p = s0; p < s1; ++p) { tstart[p] = local; local += tcnt[p]; }
        uint32_t incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        uint32_t pre = incl - local;
        for (int w = 0; w < warp; ++w) pre += wsum[w];
        for (int p = s0; p < s1; ++p) tstart[p] += pre;
        __syncthreads();
        const uint32_t nvalid = wsum[SC_TPB / 32 - 1] + 0;  // total rows of the tile with a valid key
        uint32_t total = 0;
        for (int w = 0; w < SC_TPB / 32; ++w) total += wsum[w];
        (void)nvalid;
#pragma unroll
        for (int i = 0; i < SC_R; ++i) {
            if (pp[i] < 0) continue;
            const uint32_t q = tstart[pp[i]] + rk[i];
            sval[q] = vv[i];
            skey[q] = kk[i] & (PART_GP - 1);
            spart[q] = (uint16_t)pp[i];
        }
        __syncthreads();
        for (uint32_t q = tid; q < total; q += SC_TPB) {
            const int p = spart[q];
            const uint32_t pos = cursor[p] + (q - tstart[p]);
            pkeys[pos] = skey[q];
            pvals[pos] = sval[q];
        }
        __syncthreads();
        for (int p = s0; p < s1; ++p) {
            cursor[p] += tcnt[p];
            tcnt[p] = 0;
        }
        __syncthreads();
    }
}

template <int DT, int K>
__global__ void __launch_bounds__(256, ONCHIP_MINBLOCKS)
k_part_accumulate(const int32_t *__restrict__ pkeys, const typename Fmt<DT>::V *__restrict__ pvals,
                  const int64_t *__restrict__ items, const int32_t *__restrict__ iown, int32_t *ctrl, int32_t G,
                  int32_t *pk, int64_t *pT, uint32_t *status) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int32_t s_item;
    const int n_items = ctrl[0];
    uint32_t flags = 0;
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(&ctrl[1], 1);
        __syncthreads();
        const int it = s_item;
        __syncthreads();
        if (it >= n_items) break;
        const int p = iown[it];
        const int Gi = min(PART_GP, G - p * PART_GP);
        PubArgs out{nullptr, nullptr, pk + (size_t)it * PART_GP, pT + (size_t)it * PART_GP * K};
        const SrcSingle<DT> src{{pvals}, Gi};
        accumulate_range<DT, K, true, 1>(pkeys, src, items[2 * it], items[2 * it + 1], Gi, smem, flags, out);
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && flags) atomicOr(status, flags);
}

template <int K>
__device__ __forceinline__ void realign_k(__int128 (&T)[K], int sh) {
    if (sh <= 0) return;
#pragma unroll
    for (int r = 0; r < K; ++r)
        if (r < sh) {
#pragma unroll
            for (int l = K - 1; l >= 1; --l) T[l] = T[l - 1];
            T[0] = 0;
        }
}

// Block of 32 x mw threads (mw <= MW): lane = one of 32 consecutive groups of
// a partition, warp w = items w, w+mw, ... of that partition (coalesced
// partial reads).  mw follows the expected number of items per partition.
constexpr int MW = 16;

template <int DT, int K>
__global__ void __launch_bounds__(32 * MW)
k_part_merge(int32_t G, const int64_t *__restrict__ pitem, const int32_t *__restrict__ pk,
             const int64_t *__restrict__ pT, int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D,
             typename Fmt<DT>::V *out, uint32_t *status) {
    __shared__ int32_t skm[MW][32];
    __shared__ long long sT[MW][32][K][2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, mw = blockDim.x >> 5;
    const int g = blockIdx.x * 32 + lane;
    const bool valid = g < G;
    const int gg = valid ? g : G - 1;
    const int p = gg >> PART_LOG_GP, l = gg & (PART_GP - 1);
    const int64_t i0 = pitem[p], i1 = pitem[p + 1];
    int km = 0;
    for (int64_t it = i0 + w; it < i1; it += mw) km = max(km, pk[(size_t)it * PART_GP + l]);
    skm[w][lane] = km;
    __syncthreads();
    int k = 0;
    for (int q = 0; q < mw; ++q) k = max(k, skm[q][lane]);
    __int128 T[K];
#pragma unroll
    for (int q = 0; q < K; ++q) T[q] = 0;
    for (int64_t it = i0 + w; it < i1; it += mw) {
        const int kb = pk[(size_t)it * PART_GP + l];
        __int128 Tb[K];
#pragma unroll
        for (int q = 0; q < K; ++q) Tb[q] = pT[((size_t)it * PART_GP + l) * K + q];
        realign_k<K>(Tb, k - kb);
#pragma unroll
        for (int q = 0; q < K; ++q) T[q] += Tb[q];
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
        sT[w][lane][q][0] = (long long)(uint64_t)T[q];
        sT[w][lane][q][1] = (long long)(T[q] >> 64);
    }
    __syncthreads();
    if (w != 0 || !valid) return;
#pragma unroll
    for (int q = 0; q < K; ++q) {
        T[q] = 0;
        for (int v = 0; v < mw; ++v)
            T[q] += ((__int128)sT[v][lane][q][1] << 64) + (__int128)(unsigned long long)sT[v][lane][q][0];
    }
    if (merge) {
        const int ka = acc_k[g];
        __int128 Ta[K];
#pragma unroll
        for (int q = 0; q < K; ++q) Ta[q] = join_CD<DT>(acc_C[(size_t)g * K + q], acc_D[(size_t)g * K + q]);
        const int kn = max(k, ka);
        realign_k<K>(T, kn - k);
        realign_k<K>(Ta, kn - ka);
#pragma unroll
        for (int q = 0; q < K; ++q) T[q] += Ta[q];
        k = kn;
    }
    int64_t Cc[K], Dc[K];
#pragma unroll
    for (int q = 0; q < K; ++q) split_CD<DT>(T[q], Cc[q], Dc[q]);
    if (acc_k) {
        acc_k[g] = k;
#pragma unroll
        for (int q = 0; q < K; ++q) { acc_C[(size_t)g * K + q] = Cc[q]; acc_D[(size_t)g * K + q] = Dc[q]; }
    }
    uint32_t flags = 0;
    if (out) out[g] = eq1_finalize<DT, K>(k, Cc, Dc, flags);
    if (flags) atomicOr(status, flags);
}

template <int DT, int K>
int run_partitioned(const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws, size_t ws_bytes, int merge,
                    int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out, uint32_t *status, cudaStream_t st,
                    int *launches) {
    using V = typename Fmt<DT>::V;
    if (n >= ((int64_t)1 << 32)) return -1;  // 32-bit partition cursors (callers split larger inputs)
    const Plan pl = make_plan(n, G);
    PartWs w = carve(ws, n, G, K, DT, pl);
    if (w.bytes > ws_bytes) return -1;
    const size_t hsm = 4 * (size_t)pl.P, ssm = ScatterSmem<V>::bytes(pl.P);
    if (hsm > (size_t)device_props().smem_optin) return -1;
    if (n > 0) {
        cudaFuncSetAttribute(k_part_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
        int tk = trace_begin(st);
        k_part_hist<<<pl.B, HIST_TPB, hsm, st>>>(keys, n, G, pl.P, pl.chunk, w.hist, status);
        trace_end(tk, "part_hist", st);
        ++*launches;
        tk = trace_begin(st);
        k_part_colscan<<<(pl.P + 255) / 256, 256, 0, st>>>(w.hist, pl.B, pl.P, w.ptot);
        trace_end(tk, "part_colscan", st);
        ++*launches;
    } else {
        cudaMemsetAsync(w.ptot, 0, 8 * (size_t)pl.P, st);
    }
    int tp = trace_begin(st);
    k_part_plan<<<1, 1024, 0, st>>>(w.ptot, pl.P, pl.ch, w.base, w.pitem, w.items, w.iown, w.ctrl);
    trace_end(tp, "part_plan", st);
    ++*launches;
    if (n > 0) {
        int ts = trace_begin(st);
        if (pl.P > 8 && pl.P <= 4096) {
            cudaFuncSetAttribute(k_part_scatter<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
            k_part_scatter<V><<<pl.B, SC_TPB, ssm, st>>>(keys, (const V *)vals, n, G, pl.P, pl.chunk, w.hist,
                                                         w.base, w.pkeys, (V *)w.pvals);
        } else {
            cudaFuncSetAttribute(k_part_scatter_direct<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
            k_part_scatter_direct<V><<<pl.B, HIST_TPB, hsm, st>>>(keys, (const V *)vals, n, G, pl.P, pl.chunk,
                                                                  w.hist, w.base, w.pkeys, (V *)w.pvals);
        }
        trace_end(ts, "part_scatter", st);
        ++*launches;
        // per-partition tables: Gp = 1024 groups, level sums in registers
        auto kern = k_part_accumulate<DT, K>;
        const size_t smem = onchip_smem_bytes<DT, K>(PART_GP, true);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
        if (per_sm < 1) return -1;
        const int64_t grid = std::min<int64_t>((int64_t)per_sm * device_props().sms, pl.max_items);
        int ta = trace_begin(st);
        kern<<<(unsigned)grid, 256, smem, st>>>(w.pkeys, (const V *)w.pvals, w.items, w.iown, w.ctrl, G, w.pk, w.pT,
                                                status);
        trace_end(ta, "part_accumulate", st);
        ++*launches;
    }
    int tk = trace_begin(st);
    const int64_t items_per_part = (pl.max_items + pl.P - 1) / pl.P;
    const int mw = (int)std::min<int64_t>(MW, std::max<int64_t>(1, items_per_part));
    k_part_merge<DT, K><<<(G + 31) / 32, 32 * mw, 0, st>>>(G, w.pitem, w.pk, w.pT, merge, acc_k, acc_C, acc_D,
                                                           (V *)out, status);
    trace_end(tk, "part_merge", st);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace

// one partitioning pass: histogram and direct scatter keep one 32-bit counter
// per partition in shared memory
int partition_max_groups(int, int) {
    const int64_t parts = (int64_t)device_props().smem_optin / 4;
    return (int)std::min<int64_t>(parts * PART_GP, (int64_t)1 << 30);
}

size_t partition_workspace_bytes(int64_t n, int32_t G, int K, int DT) {
    const Plan pl = make_plan(n, G);
    return carve(nullptr, n, G, K, DT, pl).bytes;
}

int launch_partitioned(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws,
                       size_t ws_bytes, int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out,
                       uint32_t *status, cudaStream_t st, int *launches) {
#define PART_CASE(dt, k)                                                                                        \
    if (DT == dt && K == k)                                                                                     \
        return run_partitioned<dt, k>(keys, vals, n, G, ws, ws_bytes, merge, acc_k, acc_C, acc_D, out, status, st, \
                                      launches);
    PART_CASE(1, 1) PART_CASE(1, 2) PART_CASE(1, 3) PART_CASE(1, 4)
    PART_CASE(0, 1) PART_CASE(0, 2) PART_CASE(0, 3) PART_CASE(0, 4)
#undef PART_CASE
    return -1;
}

}  // namespace repro
