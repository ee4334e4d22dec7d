// k_partition.cu -- high-cardinality path:
// PartitionAndAggregate (Alg. 4) on the GPU.
//
// Rows are radix-partitioned by partition id p = key >> 10 (contiguous key
// ranges of 1024 groups, one on-chip table each), most significant digit
// first, with at most 2^7 digits per pass (ParallelPartition with F = f^d,
// one pass for <= 128 partitions, two otherwise), each
// pass over SEGMENTS (the previous pass's partitions; the first pass has one):
//   1. k_seg_units    split every segment into units of <= CU rows
//   2. k_seg_hist     per unit: digit histogram (warp multisplit by ballots,
//                     per-warp counts, no shared atomics); EKEY check
//   3. k_seg_scan     per (segment, digit): unit offsets and totals
//   4. k_part_plan    exclusive scan of the totals = output bases; after the
//                     last pass also the work items of step 5 (<= CH rows,
//                     so skewed partitions are shared by many blocks)
//   5. k_seg_scatter  per unit, per 4096-row tile: warp multisplit ranks,
//                     block scan, shared staging in digit order, coalesced
//                     runs to the output (the order inside a partition is
//                     irrelevant: the accumulator is associative)
//   6. k_part_accumulate  persistent blocks pull work items and run the
//                     on-chip table code (onchip_core.cuh) on 1024 local
//                     groups, writing one partial state per (item, group)
//   7. k_part_merge   per group: max of the items' window tops, realign, add
//                     (the shared-table merge of Alg. 4 lines 6-9 via
//                     operator+=(repro)), canonicalise,
//                     Eq. 1 read-out / merge into an accumulator.
// Each group lives in exactly one partition, so no group is merged across
// partitions.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace repro {

namespace {

constexpr int PART_LOG_GP = 10;               // Gp = 1024 groups per partition
constexpr int PART_GP = 1 << PART_LOG_GP;
constexpr int64_t PART_CH = 1 << 14;          // minimum rows per work item
constexpr int SEG_TPB = 256;                 // hist / scatter blocks
constexpr int SEG_NW = SEG_TPB / 32;
#ifndef SEG_RT_DEF
#define SEG_RT_DEF 16
#endif
constexpr int SEG_RT = SEG_RT_DEF;           // rows per thread per scatter tile
#ifndef PART_IPS
#define PART_IPS 8                           // accumulate work items per SM
#endif
#ifndef SEG_HIST_BPS
#define SEG_HIST_BPS 4                       // histogram blocks per SM (2 -> 4: 0.50 -> 0.35 ms, config 3)
#endif
#ifndef SEG_RTH
#define SEG_RTH 32                           // keys per thread in flight in the histogram
#endif
#ifndef PART_HEAVY
#define PART_HEAVY 1                         // sum a partition with >= n/2 of the rows in place
#endif
#ifndef SEG_ONEPASS_BITS64
#define SEG_ONEPASS_BITS64 10                // binary64 rows: one pass up to 2^this partitions (wide above 2^8)
#endif
#ifndef SEG_ONEPASS_BITS32
#define SEG_ONEPASS_BITS32 10                // binary32 rows (wide scatter above 2^8)
#endif
constexpr int SEG_TILE = SEG_TPB * SEG_RT;   // 4096 (scatter: 8 -> 16 rows per thread: 1.98 -> 1.74 ms at 2^14 groups)
constexpr int SEG_MAX_BITS = 8;             // multisplit scatter / lane histograms: digits per pass <= 2^this
constexpr int SEG_FMAX = 1 << SEG_MAX_BITS;
static_assert(SEG_MAX_BITS <= 8, "scatter stages digits as bytes");
constexpr size_t PALIGN = 256;

inline size_t al(size_t x) { return (x + PALIGN - 1) / PALIGN * PALIGN; }

// REPRO_DEBUG=1: synchronise and report the first CUDA error after each launch
inline void dbg(const char *what) {
    static const bool on = getenv("REPRO_DEBUG") != nullptr;
    if (!on) return;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "[repro] %s: %s\n", what, cudaGetErrorString(e));
}

struct Plan {
    int64_t ch;      // rows per work item (accumulate)
    int P;           // partitions holding groups: ceil(G / 1024)
    int pbits;       // log2 of the padded partition count Pf
    int Pf;          // 1 << pbits
    int passes;      // 1 or 2
    int bits[2];     // digit bits per pass
    int shift[2];    // digit = (key >> shift) & ((1 << bits) - 1)
    int64_t cu;      // rows per unit
    int64_t max_units;
    int64_t max_items;
    int grid;        // persistent blocks of the hist / scatter kernels
    int hb;          // work items of a heavy partition summed in place
    int hgrid;       // histogram blocks
};

// Partitioning depth (f3 of SURVEY.md 8(f)): partition
// ids of up to g_onepass_bits[DT] bits are scattered in one pass, wider ones
// in two.  Defaults from the measured crossovers; settable at run
// time (repro_tune_set) and measured by repro_autotune.
int g_onepass_bits[2] = {SEG_ONEPASS_BITS32, SEG_ONEPASS_BITS64};
constexpr int SEG_ONEPASS_MAX = 10;  // the wide scatter's digit limit


// passes: 0 = by the depth setting, 1 / 2 = forced (workspace sizing)
Plan make_plan(int64_t n, int32_t G, int DT, int passes = 0) {
    Plan pl;
    pl.P = (int)(((int64_t)G + PART_GP - 1) >> PART_LOG_GP);
    pl.pbits = 0;
    while ((1 << pl.pbits) < pl.P) ++pl.pbits;
    pl.Pf = 1 << pl.pbits;
    bool one = pl.pbits <= g_onepass_bits[DT == 1];
    if (passes == 1) one = pl.pbits <= SEG_ONEPASS_MAX;
    if (passes == 2) one = pl.pbits < 2;
    if (pl.pbits > 2 * SEG_MAX_BITS) one = false;
    if (one) {
        pl.passes = 1;
        pl.bits[0] = pl.pbits;
        pl.shift[0] = PART_LOG_GP;
        pl.bits[1] = 0;
        pl.shift[1] = 0;
    } else {
        pl.passes = 2;
        pl.bits[1] = (pl.pbits + 1) / 2;
        pl.bits[0] = pl.pbits - pl.bits[1];
        pl.shift[0] = PART_LOG_GP + pl.bits[1];
        pl.shift[1] = PART_LOG_GP;
    }
    const int sms = device_props().sms;
    pl.cu = std::max<int64_t>(1 << 14, (n + 8 * sms - 1) / (8 * sms));
    pl.max_units = (n + pl.cu - 1) / pl.cu + (1 << pl.bits[0]) + 1;
    pl.grid = (int)std::max<int64_t>(1, std::min<int64_t>(2 * sms, pl.max_units));
    pl.hgrid = (int)std::max<int64_t>(1, std::min<int64_t>(SEG_HIST_BPS * sms, pl.max_units));
    // work items: ~PART_IPS per SM over the whole input, at least PART_CH rows
    pl.ch = std::max<int64_t>(PART_CH, (n + PART_IPS * sms - 1) / (PART_IPS * sms));
    pl.hb = 2 * sms;
    pl.max_items = (n + pl.ch - 1) / pl.ch + pl.Pf + pl.hb;
    return pl;
}

struct PartWs {
    int32_t *pkeys;   // final partitioned rows (local keys)
    void *pvals;
    int32_t *akeys;   // first-pass output of a two-pass plan (full keys)
    void *avals;
    uint32_t *hist;   // [max_units][2^bits] unit offsets per digit
    int64_t *units;   // [max_units][2] row range
    int32_t *useg;    // [max_units] segment of each unit
    int32_t *ufirst;  // [2^bits0 + 2] first unit of each segment (+ count)
    int64_t *ptot;    // [Pf]    partition sizes
    int64_t *base;    // [Pf+1]  first row of each partition
    int64_t *pitem;   // [Pf+1]  first work item of each partition
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
    const int fmax = 1 << std::max(pl.bits[0], pl.bits[1]);
    w.pkeys = (int32_t *)take(4 * (size_t)n + 16);
    w.pvals = take(vsz * (size_t)n + 16);
    if (pl.passes == 2) {
        w.akeys = (int32_t *)take(4 * (size_t)n + 16);
        w.avals = take(vsz * (size_t)n + 16);
    }
    w.hist = (uint32_t *)take(4 * (size_t)pl.max_units * fmax);  // fmax <= 2^SEG_ONEPASS_BITS
    w.units = (int64_t *)take(16 * (size_t)pl.max_units);
    w.useg = (int32_t *)take(4 * (size_t)pl.max_units);
    w.ufirst = (int32_t *)take(4 * ((size_t)(1 << pl.bits[0]) + 2));
    w.ptot = (int64_t *)take(8 * (size_t)pl.Pf);
    w.base = (int64_t *)take(8 * ((size_t)pl.Pf + 1));
    w.pitem = (int64_t *)take(8 * ((size_t)pl.Pf + 1));
    w.items = (int64_t *)take(16 * (size_t)pl.max_items);
    w.iown = (int32_t *)take(4 * (size_t)pl.max_items);
    w.ctrl = (int32_t *)take(16);
    w.pk = (int32_t *)take(4 * (size_t)pl.max_items * PART_GP);
    w.pT = (int64_t *)take(8 * (size_t)pl.max_items * PART_GP * K);
    w.bytes = o;
    return w;
}

// ---- segmented radix passes ------------------------------------------------

// Units: segment s = rows [base[s], base[s+1]) (base == nullptr: one segment
// [0, n)) split into ceil(len / cu) units.  Single block.
__global__ void __launch_bounds__(1024) k_seg_units(const int64_t *base, int S, int64_t n, int64_t cu, int64_t *units,
                                                    int32_t *useg, int32_t *ufirst) {
    __shared__ int32_t wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (S + 1023) / 1024;
    const int s0 = min(tid * per, S), s1 = min(s0 + per, S);
    auto seg = [&](int s, int64_t &a, int64_t &b) {
        a = base ? base[s] : 0;
        b = base ? base[s + 1] : n;
    };
    int cnt = 0;
    for (int s = s0; s < s1; ++s) {
        int64_t a, b;
        seg(s, a, b);
        cnt += (int)((b - a + cu - 1) / cu);
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int u = incl - cnt;
    for (int w = 0; w < warp; ++w) u += wsum[w];
    for (int s = s0; s < s1; ++s) {
        int64_t a, b;
        seg(s, a, b);
        ufirst[s] = u;
        for (int64_t r = a; r < b; r += cu, ++u) {
            units[2 * u] = r;
            units[2 * u + 1] = min(b, r + cu);
            useg[u] = s;
        }
    }
    if (tid == 1023) {
        ufirst[S] = u;      // total units
        ufirst[S + 1] = u;
    }
}

// Warp multisplit of one 32-row slot: lanes whose `ok` is set and whose digit
// d (bits bits) is equal form one peer set (mask from one ballot per bit);
// returns the peer mask.
__device__ __forceinline__ uint32_t peers_of(int d, int bits, bool ok) {
    uint32_t m = __ballot_sync(0xffffffffu, ok);
    for (int b = 0; b < bits; ++b) {
        const bool bit = (d >> b) & 1;
        const uint32_t bb = __ballot_sync(0xffffffffu, bit);
        m &= bit ? bb : ~bb;
    }
    return ok ? m : 0u;
}

// Digit histogram per unit.  F <= 32: one private counter row per lane
// (counter [warp][d][lane], always bank = lane: plain load-add-store, no
// atomics, no conflicts); F > 32: per-warp histograms with shared atomics.
// Both are summed over lanes / warps at the end of the unit.  The first pass
// also checks the keys against [0, G).
__global__ void __launch_bounds__(SEG_TPB)
k_seg_hist(const int32_t *__restrict__ keys, const int64_t *__restrict__ units, const int32_t *__restrict__ ufirst,
           int S, int shift, int bits, int32_t G, int check, uint32_t *hist, uint32_t *status) {
    __shared__ uint32_t h[SEG_NW * 32 * 32];  // lane rows (F <= 32) or [NW][F] (F > 32): 32 KB
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int F = 1 << bits;
    const bool lanes = F <= 32;
    const int nunits = ufirst[S];
    uint32_t *hw = lanes ? h + warp * 32 * 32 : h + warp * F;
    uint32_t bad = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        for (int i = tid; i < SEG_NW * 32 * 32; i += SEG_TPB) h[i] = 0;
        __syncthreads();
        const int64_t a = units[2 * u], b = units[2 * u + 1];
        for (int64_t r0 = a + warp * 32 * SEG_RTH; r0 < b; r0 += SEG_NW * 32 * SEG_RTH) {
            int kk[SEG_RTH];  // SEG_RTH warp slots in flight per thread
#pragma unroll
            for (int j = 0; j < SEG_RTH; ++j) {
                const int64_t r = r0 + j * 32 + lane;
                kk[j] = r < b ? __ldg(keys + r) : -1;
                if (check && r < b && (uint32_t)kk[j] >= (uint32_t)G) bad = FLAG_EKEY;
            }
#pragma unroll
            for (int j = 0; j < SEG_RTH; ++j) {
                if ((uint32_t)kk[j] < (uint32_t)G) {
                    const int d = (kk[j] >> shift) & (F - 1);
                    if (lanes) hw[d * 32 + lane] += 1u;
                    else atomicAdd(&hw[d], 1u);
                }
            }
        }
        __syncthreads();
        for (int d = tid; d < F; d += SEG_TPB) {
            uint32_t t = 0;
            if (lanes) {
                for (int w = 0; w < SEG_NW; ++w)
                    for (int l = 0; l < 32; ++l) t += h[w * 1024 + d * 32 + ((l + d) & 31)];
            } else {
                for (int w = 0; w < SEG_NW; ++w) t += h[w * F + d];
            }
            hist[(size_t)u * F + d] = t;
        }
        __syncthreads();
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicOr(status, bad);
}

// per (segment s, digit d), one block each: hist[u][d] <- rows of digit d in
// the units of s before u (block-wide scan over the units, 256 at a time);
// ptot[s * F + d] <- total
__global__ void __launch_bounds__(256) k_seg_scan(uint32_t *hist, const int32_t *__restrict__ ufirst, int bits,
                                                  int64_t *ptot) {
    __shared__ int64_t wsum[8];
    const int F = 1 << bits;
    const int s = blockIdx.x / F, d = blockIdx.x - s * F;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int u0 = ufirst[s], u1 = ufirst[s + 1];
    int64_t run = 0;
    for (int c = u0; c < u1; c += 256) {
        const int u = c + tid;
        const int64_t v = u < u1 ? hist[(size_t)u * F + d] : 0;
        int64_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int64_t pre = run + incl - v, tot = 0;
        for (int w = 0; w < 8; ++w) {
            if (w < warp) pre += wsum[w];
            tot += wsum[w];
        }
        if (u < u1) hist[(size_t)u * F + d] = (uint32_t)pre;
        run += tot;
        __syncthreads();
    }
    if (tid == 0) ptot[blockIdx.x] = run;
}

// single block: base[] = exclusive scan of ptot, pitem[] = exclusive scan of
// the items per partition, then the item table.  heavy_ok (last pass of a
// one-pass plan, n >= 2^20): a partition holding >= n/2 of the rows (the
// heaviest; ties: lowest id) is not scattered -- its rows keep no space in the
// output (ctrl[2] = its id, the scatter skips them) and it gets HB items over
// the ORIGINAL row range [0, n), which k_part_accumulate reads through a
// partition filter (skewed keys: the hot partition is summed in place).
// Break-even: scattering a partition costs a write and a re-read of its rows
// (2 n_h row bytes), the in-place sum re-reads the whole input (n row bytes).
__global__ void __launch_bounds__(1024) k_part_plan(const int64_t *ptot, int P, int64_t chunk_rows, int64_t *base,
                                                    int64_t *pitem, int64_t *items, int32_t *iown, int32_t *ctrl,
                                                    int heavy_ok, int64_t n, int hb) {
    __shared__ int64_t wsum[2][32];
    __shared__ unsigned long long s_best;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (P + 1023) / 1024;
    const int p0 = min(tid * per, P), p1 = min(p0 + per, P);
    if (tid == 0) s_best = 0ull;
    __syncthreads();
    if (heavy_ok) {
        unsigned long long best = 0ull;  // (rows << 20) | (2^20 - 1 - p): max rows, then lowest p
        for (int p = p0; p < p1; ++p)
            best = max(best, ((unsigned long long)ptot[p] << 20) | (unsigned long long)((1 << 20) - 1 - p));
        atomicMax(&s_best, best);
    }
    __syncthreads();
    int heavy = -1;
    if (heavy_ok && (int64_t)(s_best >> 20) * 2 >= n) heavy = (1 << 20) - 1 - (int)(s_best & ((1u << 20) - 1));
    auto rows_of = [&](int p) { return p == heavy ? (int64_t)0 : ptot[p]; };
    auto items_of = [&](int p) { return p == heavy ? (int64_t)hb : (ptot[p] + chunk_rows - 1) / chunk_rows; };
    int64_t rows = 0, its = 0;
    for (int p = p0; p < p1; ++p) {
        rows += rows_of(p);
        its += items_of(p);
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
        const int64_t c = items_of(p);
        if (p == heavy) {
            // chunks of a multiple of 256 rows: every item starts 16-byte aligned (TMA ring)
            const int64_t ch = ((n + hb - 1) / hb + 255) / 256 * 256;
            for (int64_t i = 0; i < c; ++i) {
                items[2 * (pi + i)] = min(n, i * ch);
                items[2 * (pi + i) + 1] = min(n, (i + 1) * ch);
                iown[pi + i] = p;
            }
        } else {
            for (int64_t i = 0; i < c; ++i) {
                items[2 * (pi + i)] = pr + i * chunk_rows;
                items[2 * (pi + i) + 1] = min(pr + (i + 1) * chunk_rows, pr + ptot[p]);
                iown[pi + i] = p;
            }
        }
        pr += rows_of(p);
        pi += c;
    }
    if (tid == 1023) {
        base[P] = pr;
        pitem[P] = pi;
        ctrl[0] = (int32_t)pi;
        ctrl[1] = 0;
        ctrl[2] = heavy;
    }
}

// Scatter one pass: per unit (persistent blocks), per tile of SEG_TILE rows:
// every row's rank among the tile's rows of its digit from the warp
// multisplit (per-warp running counts, no shared atomics), a block scan over
// (digit, warp), staging in digit order in shared memory, then coalesced runs
// to cursor[d] (output base of (segment, digit) + the unit's offset).  LOCAL:
// write the key within its 1024-group partition (last pass).
template <typename V>
__global__ void __launch_bounds__(SEG_TPB)
k_seg_scatter(const int32_t *__restrict__ ikeys, const V *__restrict__ ivals, const int64_t *__restrict__ units,
              const int32_t *__restrict__ useg, const int32_t *__restrict__ ufirst, int S, int shift, int bits,
              int32_t G, int local, const uint32_t *__restrict__ hist, const int64_t *__restrict__ obase,
              int32_t *__restrict__ okeys, V *__restrict__ ovals, const int32_t *__restrict__ ctrl) {
    constexpr int TPB = SEG_TPB, NW = SEG_NW, RT = SEG_RT, TILE = SEG_TILE;
    const int heavy = local ? ctrl[2] : -1;  // heavy partition: summed in place, not scattered
    extern __shared__ __align__(16) unsigned char sm[];
    V *sval = reinterpret_cast<V *>(sm);                          // [TILE]
    int32_t *skey = reinterpret_cast<int32_t *>(sval + TILE);     // [TILE]
    uint8_t *sdig = reinterpret_cast<uint8_t *>(skey + TILE);     // [TILE]
    uint32_t *wh = reinterpret_cast<uint32_t *>(sdig + TILE);     // [NW][FMAX] running counts, then offsets
    uint32_t *tot = wh + NW * SEG_FMAX;                           // [FMAX] tile totals
    uint32_t *tstart = tot + SEG_FMAX;                            // [FMAX] tile start of each digit
    int64_t *cursor = reinterpret_cast<int64_t *>(tstart + SEG_FMAX);  // [FMAX]
    uint32_t *wsc = reinterpret_cast<uint32_t *>(cursor + SEG_FMAX);   // [32] scan scratch
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int F = 1 << bits;
    const int nunits = ufirst[S];
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int s = useg[u];
        for (int d = tid; d < F; d += TPB) cursor[d] = obase[(size_t)s * F + d] + hist[(size_t)u * F + d];
        const int64_t a = units[2 * u], b = units[2 * u + 1];
        for (int64_t t0 = a; t0 < b; t0 += TILE) {
            for (int d = lane; d < F; d += 32) wh[warp * SEG_FMAX + d] = 0;
            __syncwarp();
            int kk[RT], dd[RT];
            uint32_t rk[RT];
            V vv[RT];
#pragma unroll
            for (int j = 0; j < RT; ++j) {
                const int64_t r = t0 + (int64_t)(j * NW + warp) * 32 + lane;  // warp-contiguous 32-row slots
                kk[j] = -1;
                vv[j] = V(0);
                if (r < b) {
                    kk[j] = __ldg(ikeys + r);
                    vv[j] = __ldg(ivals + r);
                }
            }
#pragma unroll
            for (int j = 0; j < RT; ++j) {
                bool valid = (uint32_t)kk[j] < (uint32_t)G;
                dd[j] = valid ? (kk[j] >> shift) & (F - 1) : 0;
                valid = valid && dd[j] != heavy;
                const uint32_t m = peers_of(dd[j], bits, valid);
                const uint32_t before = valid ? wh[warp * SEG_FMAX + dd[j]] : 0u;
                rk[j] = valid ? before + __popc(m & ((1u << lane) - 1u)) : 0xFFFFFFFFu;
                __syncwarp();
                if (valid && (m & ((1u << lane) - 1u)) == 0u) wh[warp * SEG_FMAX + dd[j]] = before + __popc(m);
                __syncwarp();
            }
            __syncthreads();
            // exclusive scan over (digit, warp): wh[w][d] <- tile offset of
            // warp w's rows of digit d; tstart[d], tot[d]
            const int per = (F * NW + TPB - 1) / TPB;  // entries per thread, digit-major order
            const int e0 = min(tid * per, F * NW), e1 = min(e0 + per, F * NW);
            uint32_t loc = 0;
            for (int e = e0; e < e1; ++e) loc += wh[(e % NW) * SEG_FMAX + e / NW];
            uint32_t incl = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wsc[warp] = incl;
            __syncthreads();
            uint32_t run = incl - loc;
            for (int w = 0; w < warp; ++w) run += wsc[w];
            for (int e = e0; e < e1; ++e) {
                const int d = e / NW, w = e % NW;
                const uint32_t c = wh[w * SEG_FMAX + d];
                if (w == 0) tstart[d] = run;
                wh[w * SEG_FMAX + d] = run;
                run += c;
            }
            __syncthreads();
            uint32_t ntile = 0;
            for (int w = 0; w < NW; ++w) ntile += wsc[w];
            for (int d = tid; d < F; d += TPB) tot[d] = (d + 1 < F ? tstart[d + 1] : ntile) - tstart[d];
#pragma unroll
            for (int j = 0; j < RT; ++j) {
                if (rk[j] == 0xFFFFFFFFu) continue;
                const uint32_t q = wh[warp * SEG_FMAX + dd[j]] + rk[j];
                sval[q] = vv[j];
                skey[q] = local ? (kk[j] & (PART_GP - 1)) : kk[j];
                sdig[q] = (uint8_t)dd[j];
            }
            __syncthreads();
            for (uint32_t q = tid; q < ntile; q += TPB) {
                const int d = sdig[q];
                const int64_t pos = cursor[d] + (q - tstart[d]);
                okeys[pos] = skey[q];
                ovals[pos] = sval[q];
            }
            __syncthreads();
            for (int d = tid; d < F; d += TPB) cursor[d] += tot[d];
            __syncthreads();
        }
    }
}

// Wide-fan-out scatter (F > 2^SEG_MAX_BITS, single pass): ranks inside the
// tile from shared-memory atomics on per-digit counters (fine when F is large:
// few lanes share a counter), block scan over the digits, staging in digit
// order, coalesced runs to the output.
constexpr int WS_TPB = 512;
// rows per thread per tile: longer output runs per digit at the wide fan-out
// (measured: binary64 512-way 3.71 / 3.11 / 2.86 ms at 8 / 12 / 16 rows;
// binary32 config 3 1.23 / 1.12 / 1.49 ms)
template <typename V>
constexpr int ws_r() { return sizeof(V) == 8 ? 16 : 12; }
template <typename V>
constexpr int ws_tile() { return WS_TPB * ws_r<V>(); }

template <typename V>
constexpr size_t seg_scatter_wide_smem(int F) {
    return (size_t)12 * F + 64 * 4 + (size_t)ws_tile<V>() * (sizeof(V) + 4 + 2) + 64;
}

template <typename V>
__global__ void __launch_bounds__(WS_TPB)
k_seg_scatter_wide(const int32_t *__restrict__ ikeys, const V *__restrict__ ivals, const int64_t *__restrict__ units,
                   const int32_t *__restrict__ useg, const int32_t *__restrict__ ufirst, int S, int shift, int bits,
                   int32_t G, int local, const uint32_t *__restrict__ hist, const int64_t *__restrict__ obase,
                   int32_t *__restrict__ okeys, V *__restrict__ ovals, const int32_t *__restrict__ ctrl) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int F = 1 << bits;
    const int heavy = local ? ctrl[2] : -1;  // heavy partition: summed in place, not scattered
    uint32_t *cursor = reinterpret_cast<uint32_t *>(sm);  // [F] next output row (n < 2^32)
    uint32_t *tcnt = cursor + F;                           // [F] rows of the tile per digit
    uint32_t *tstart = tcnt + F;                           // [F] tile-local start
    uint32_t *wsum = tstart + F;                           // [32] scan scratch
    V *sval = reinterpret_cast<V *>(sm + (((size_t)12 * F + 64 * 4 + 15) & ~(size_t)15));
    constexpr int WS_R = ws_r<V>(), WS_TILE = ws_tile<V>();
    int32_t *skey = reinterpret_cast<int32_t *>(sval + WS_TILE);
    uint16_t *sdig = reinterpret_cast<uint16_t *>(skey + WS_TILE);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cper = (F + WS_TPB - 1) / WS_TPB;
    const int s0 = min(tid * cper, F), s1 = min(s0 + cper, F);
    const int nunits = ufirst[S];
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int sg = useg[u];
        for (int d = tid; d < F; d += WS_TPB) {
            cursor[d] = (uint32_t)(obase[(size_t)sg * F + d] + hist[(size_t)u * F + d]);
            tcnt[d] = 0;
        }
        __syncthreads();
        const int64_t a = units[2 * u], b = units[2 * u + 1];
        for (int64_t tb = a; tb < b; tb += WS_TILE) {
            int kk[WS_R], dd[WS_R];
            uint32_t rk[WS_R];
            V vv[WS_R];
#pragma unroll
            for (int i = 0; i < WS_R; ++i) {
                const int64_t r = tb + (int64_t)i * WS_TPB + tid;
                kk[i] = -1;
                vv[i] = V(0);
                if (r < b) {
                    kk[i] = __ldg(ikeys + r);
                    vv[i] = __ldg(ivals + r);
                }
            }
#pragma unroll
            for (int i = 0; i < WS_R; ++i) {
                dd[i] = (uint32_t)kk[i] < (uint32_t)G ? (kk[i] >> shift) & (F - 1) : -1;
                if (dd[i] == heavy) dd[i] = -1;
                rk[i] = dd[i] >= 0 ? atomicAdd(&tcnt[dd[i]], 1u) : 0u;
            }
            __syncthreads();
            uint32_t loc = 0;
            for (int d = s0; d < s1; ++d) { tstart[d] = loc; loc += tcnt[d]; }
            uint32_t incl = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            uint32_t pre = incl - loc;
            for (int w = 0; w < warp; ++w) pre += wsum[w];
            for (int d = s0; d < s1; ++d) tstart[d] += pre;
            __syncthreads();
            uint32_t total = 0;
            for (int w = 0; w < WS_TPB / 32; ++w) total += wsum[w];
#pragma unroll
            for (int i = 0; i < WS_R; ++i) {
                if (dd[i] < 0) continue;
                const uint32_t q = tstart[dd[i]] + rk[i];
                sval[q] = vv[i];
                skey[q] = local ? (kk[i] & (PART_GP - 1)) : kk[i];
                sdig[q] = (uint16_t)dd[i];
            }
            __syncthreads();
            for (uint32_t q = tid; q < total; q += WS_TPB) {
                const int d = sdig[q];
                const uint32_t pos = cursor[d] + (q - tstart[d]);
                okeys[pos] = skey[q];
                ovals[pos] = sval[q];
            }
            __syncthreads();
            for (int d = s0; d < s1; ++d) {
                cursor[d] += tcnt[d];
                tcnt[d] = 0;
            }
            __syncthreads();
        }
    }
}

template <typename V>
constexpr size_t seg_scatter_smem() {
    return (size_t)SEG_TILE * (sizeof(V) + 4 + 1) + 4 * (size_t)SEG_NW * SEG_FMAX + 8 * (size_t)SEG_FMAX +
           8 * (size_t)SEG_FMAX + 4 * 32 + 64;
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
        if (p == ctrl[2]) continue;  // heavy partition: k_part_heavy sums it in place
        const SrcSingle<DT> src{{pvals}, Gi};
        accumulate_range<DT, K, true, 1>(pkeys, src, items[2 * it], items[2 * it + 1], Gi, smem, flags, out);
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && flags) atomicOr(status, flags);
}

// The heavy partition (k_part_plan): block b sums the rows of item
// pitem[h] + b -- a range of the ORIGINAL columns -- through the partition
// filter with the TMA-fed on-chip code, writing that item's partial states.
// Launched unconditionally; blocks exit at once when there is no heavy
// partition (the decision is on the device).
template <int DT, int K, bool TMA>
__global__ void __launch_bounds__(256, ONCHIP_MINBLOCKS)
k_part_heavy(const int32_t *__restrict__ keys, const typename Fmt<DT>::V *__restrict__ vals,
             const int64_t *__restrict__ items, const int64_t *__restrict__ pitem, const int32_t *__restrict__ ctrl,
             int32_t G, int32_t *pk, int64_t *pT, uint32_t *status) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int h = ctrl[2];
    if (h < 0) return;
    const int64_t it = pitem[h] + blockIdx.x;
    if (it >= pitem[h + 1]) return;
    const int Gi = min(PART_GP, G - h * PART_GP);
    uint32_t flags = 0;
    PubArgs out{nullptr, nullptr, pk + (size_t)it * PART_GP, pT + (size_t)it * PART_GP * K};
    const SrcFiltered<DT> src{{vals}, Gi, h};
    accumulate_range<DT, K, true, 1, TMA>(keys, src, items[2 * it], items[2 * it + 1], Gi, smem, flags, out);
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
    const Plan pl = make_plan(n, G, DT);
    PartWs w = carve(ws, n, G, K, DT, pl);
    if (w.bytes > ws_bytes) return -1;
    constexpr size_t ssm = seg_scatter_smem<V>();
    if (ssm > (size_t)device_props().smem_optin) return -1;
    if (n == 0) {
        cudaMemsetAsync(w.ptot, 0, 8 * (size_t)pl.Pf, st);
        int tp = trace_begin(st);
        k_part_plan<<<1, 1024, 0, st>>>(w.ptot, pl.Pf, pl.ch, w.base, w.pitem, w.items, w.iown, w.ctrl, 0, n,
                                        pl.hb);
        trace_end(tp, "part_plan", st);
            dbg("part_plan");
        ++*launches;
    } else {
        cudaFuncSetAttribute(k_seg_scatter<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
        const int32_t *ik = keys;
        const V *iv = (const V *)vals;
        int S = 1;
        for (int pass = 0; pass < pl.passes; ++pass) {
            const bool last = pass + 1 == pl.passes;
            const int bits = pl.bits[pass], F = 1 << bits;
            int32_t *ok = last ? w.pkeys : w.akeys;
            V *ov = (V *)(last ? w.pvals : w.avals);
            int tk = trace_begin(st);
            k_seg_units<<<1, 1024, 0, st>>>(pass == 0 ? nullptr : w.base, S, n, pl.cu, w.units, w.useg, w.ufirst);
            ++*launches;
            k_seg_hist<<<pl.hgrid, SEG_TPB, 0, st>>>(ik, w.units, w.ufirst, S, pl.shift[pass], bits, G, pass == 0,
                                                     w.hist, status);
            ++*launches;
            k_seg_scan<<<S * F, 256, 0, st>>>(w.hist, w.ufirst, bits, w.ptot);
            ++*launches;
            const int heavy_ok = PART_HEAVY && pl.passes == 1 && n >= (1 << 20);
            k_part_plan<<<1, 1024, 0, st>>>(w.ptot, S * F, pl.ch, w.base, w.pitem, w.items, w.iown, w.ctrl, heavy_ok,
                                            n, pl.hb);
            ++*launches;
            trace_end(tk, "part_hist", st);
            dbg("part_hist");
            tk = trace_begin(st);
            if (bits <= SEG_MAX_BITS) {
                k_seg_scatter<V><<<pl.grid, SEG_TPB, ssm, st>>>(ik, iv, w.units, w.useg, w.ufirst, S, pl.shift[pass],
                                                               bits, G, last ? 1 : 0, w.hist, w.base, ok, ov, w.ctrl);
            } else {
                const size_t wsm = seg_scatter_wide_smem<V>(F);
                cudaFuncSetAttribute(k_seg_scatter_wide<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
                k_seg_scatter_wide<V><<<pl.grid, WS_TPB, wsm, st>>>(ik, iv, w.units, w.useg, w.ufirst, S,
                                                                    pl.shift[pass], bits, G, last ? 1 : 0, w.hist,
                                                                    w.base, ok, ov, w.ctrl);
            }
            trace_end(tk, "part_scatter", st);
            dbg("part_scatter");
            ++*launches;
            ik = ok;
            iv = ov;
            S *= F;
        }
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
            dbg("part_accumulate");
        ++*launches;
        if (PART_HEAVY && pl.passes == 1 && n >= (1 << 20)) {
            // the heavy partition (if the plan found one) straight from the input
            const bool tma = ((((uintptr_t)keys) | ((uintptr_t)vals)) & 15) == 0;
            auto hk = tma ? k_part_heavy<DT, K, true> : k_part_heavy<DT, K, false>;
            const size_t hsm = onchip_smem_bytes<DT, K>(PART_GP, true, tma);
            cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
            int th = trace_begin(st);
            hk<<<pl.hb, 256, hsm, st>>>(keys, (const V *)vals, w.items, w.pitem, w.ctrl, G, w.pk, w.pT, status);
            trace_end(th, "part_heavy", st);
            dbg("part_heavy");
            ++*launches;
        }
    }
    int tk = trace_begin(st);
    const int64_t items_per_part = (pl.max_items + pl.P - 1) / pl.P;
    const int mw = (int)std::min<int64_t>(MW, std::max<int64_t>(1, items_per_part));
    k_part_merge<DT, K><<<(G + 31) / 32, 32 * mw, 0, st>>>(G, w.pitem, w.pk, w.pT, merge, acc_k, acc_C, acc_D,
                                                           (V *)out, status);
    trace_end(tk, "part_merge", st);
            dbg("part_merge");
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace

// at most two passes of <= 2^8 digits: 2^16 partitions of 1024 groups
int partition_max_groups(int, int) { return 1 << (2 * SEG_MAX_BITS + PART_LOG_GP); }

int partition_onepass_bits(int DT) { return g_onepass_bits[DT == 1]; }
int set_partition_onepass_bits(int DT, int bits) {
    if (bits < 1 || bits > SEG_ONEPASS_MAX) return -1;
    g_onepass_bits[DT == 1] = bits;
    return 0;
}

// sized for both depths where both are possible, so that a depth change
// (repro_tune_set / repro_autotune) never outgrows a caller's workspace
size_t partition_workspace_bytes(int64_t n, int32_t G, int K, int DT) {
    size_t b = carve(nullptr, n, G, K, DT, make_plan(n, G, DT)).bytes;
    for (int p = 1; p <= 2; ++p) {
        const Plan pl = make_plan(n, G, DT, p);
        if (pl.passes == 1 && pl.pbits > SEG_ONEPASS_MAX) continue;
        b = std::max(b, carve(nullptr, n, G, K, DT, pl).bytes);
    }
    return b;
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
