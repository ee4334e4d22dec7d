// k_table.cu -- the on-chip GroupBy-SUM kernel for one value column and up to
// a few thousand groups.
//
// One persistent block per contiguous row range keeps a table of 32-bit LIMB
// COUNTERS in shared memory (word-major: counter w of group g at w*GQ + g, so
// a warp's random groups spread over the banks) and nothing else per group
// but its window top.  Rows stream straight from HBM in 16-byte vectors (a
// quad of 4 rows per thread, the next step's quads in flight while this one
// is deposited).  Each row's K digits (Alg. 1 lines 10-16)
// are read from the bits of x (+) E_l (Extractors, onchip_core.cuh) and added
// with native 32-bit shared atomics (binary64: two balanced 20-bit limbs per
// digit, binary32: one).
//
// Every level sum leaves the block through the ABSOLUTE-LEVEL slot table
// (kglob, slots): a row's digit at level j does not depend on the window it
// was computed in (digits above k* are zero), so a block may publish a
// group's counters at any window w >= the k* of the rows they hold and the
// fold kernel reads the K slots under the group's global top (k_state.cu).
// That removes all per-block level bookkeeping from the hot loop:
//   * carry renormalisation (Alg. 1 lines 17-21, deferred as in Alg. 2's NB
//     blocking): every deposit atomic returns the counter's
//     old value; a thread that sees |old| >= 2^29 swaps the counter with zero
//     (atom.exch) and adds what it took to the slot table.  At most one batch
//     per thread lands between the first such observation and the swap, so a
//     counter stays below 2^29 + TPB * 4 * 2^19 < 2^31.  No block barrier;
//   * level shifts (Alg. 1 lines 3-9): while the groups'
//     tops differ, tiles are processed block-synchronously (per-row k*,
//     shared atomicMax, and a group whose top rises publishes its counters at
//     the old window and restarts them at the new one -- the paper's
//     demotion, exact through the absolute slots).  Once every group of the
//     block has the same top kuni, the block streams without barriers: a row
//     with k* > kuni is deposited straight into the slot table at its own
//     window k* (and raises the group's global top), which is exact for the
//     same reason.
//   * band mode (the > 2048-group kernel only, Table XB = 1): a block whose
//     groups still differ in top after the first tile streams with every row
//     at its own window over K + 1 levels (table_core.cuh) until every group
//     reached the top.  The <= 2048-group kernels stay block-synchronous in
//     that case: compiled into their loop, the band mode cost the uniform
//     mode -- config 1 -- 4-5% (registers).
// Rows with a key outside [0, G) or a NaN/Inf/ERANGE value set the status
// bits (precedence EKEY > EDOM > ERANGE on read) and deposit nothing.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"
#include "table_core.cuh"

#include <algorithm>

namespace repro {

namespace {

#ifndef TAB_QPT
#define TAB_QPT 2  // quads (4 rows) per thread per step (256-thread kernels); the next step's are in flight
#endif
#ifndef TAB_QPT512
#define TAB_QPT512 1  // the same for the one-block-per-SM (> 2048 groups) kernels
#endif
#ifndef TAB_BIGTPB
#define TAB_BIGTPB 512  // threads of the one-block-per-SM (> 2048 groups) kernels (384, with 1 or 2 quads: slower)
#endif
#ifndef TAB_L2PF
#define TAB_L2PF 0  // (measured slower: 0.419 -> 0.461 ms at 3 steps) steps ahead whose rows lane 0 of each warp prefetches into L2 (0: off)
#endif

#ifndef TAB_OBS2
#define TAB_OBS2 1  // 1: counters observed on every other quad only (red.shared in between; TPB <= 256)
#endif  // (config 1, 2^27 rows: QPT 1 / OBS2 0 0.419 ms, QPT 2 + OBS2 0.406 ms; each alone is slower)
#ifndef TAB_MINB256
#define TAB_MINB256 2  // resident 256-thread blocks per SM the register budget is sized for
#endif

#if TAB_DEBUG
__device__ unsigned long long g_tab_modes[3];
#endif

template <int DT, int K, int TPB, bool VEC, int GQC, int XB>
__global__ void __launch_bounds__(TPB, TPB == 256 ? TAB_MINB256 : 1)
k_table(const int32_t *__restrict__ keys, const typename Fmt<DT>::V *__restrict__ vals, int64_t n, int32_t G,
        int64_t chunk, int32_t *__restrict__ kglob, unsigned long long *__restrict__ slots,
        uint32_t *__restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_mm[TAB_MM];
    const int tid = threadIdx.x;
    const int64_t row0 = (int64_t)blockIdx.x * chunk;
    const int64_t row1 = min(n, row0 + chunk);
    if (row0 >= row1) return;
    Table<DT, K, TPB, GQC, false, XB> tab(smem, s_mm, G, 0, kglob, slots);
    tab.clear();
    uint32_t flags = 0;
    __syncthreads();

    // whole quads [row0, row0 + 4 nq), then a tail of < 4 rows
    const int64_t nq = (row1 - row0) >> 2;
    // software pipeline: the next step's quads are in flight while this
    // step's are deposited (quad i of step s: q = (s QPT + i) TPB + tid)
    constexpr int QPT = TPB == 256 ? TAB_QPT : TAB_QPT512;
    QuadT<DT> nxt[QPT];
    const int64_t steps = (nq + TPB * QPT - 1) / (TPB * QPT);
#pragma unroll
    for (int i = 0; i < QPT; ++i)
        if (i * TPB + tid < nq) load_quad<DT, VEC>(keys, vals, row0 + 4 * (int64_t)(i * TPB + tid), nxt[i]);
    // one step: the next step's quads are issued, this step's deposited
    auto step = [&](int64_t s, auto &&deposit) {
        QuadT<DT> cur[QPT];
#pragma unroll
        for (int i = 0; i < QPT; ++i) cur[i] = nxt[i];
        const int64_t q0 = s * TPB * QPT + tid;
#pragma unroll
        for (int i = 0; i < QPT; ++i) {
            const int64_t qn = q0 + (int64_t)(QPT + i) * TPB;
            if (qn < nq) load_quad<DT, VEC>(keys, vals, row0 + 4 * qn, nxt[i]);
        }
        if (TAB_L2PF > 0 && VEC && (tid & 31) == 0) {
            // deeper memory-level parallelism without registers: the warp's
            // rows TAB_L2PF steps ahead (contiguous: 32 quads per quad slot)
            // are pulled into L2 by bulk prefetches
#pragma unroll
            for (int i = 0; i < QPT; ++i) {
                const int64_t qp = q0 + (int64_t)(TAB_L2PF * QPT + i) * TPB;
                if (qp + 32 <= nq) {
                    const int64_t r = row0 + 4 * qp;
                    l2_prefetch(keys + r, 128 * 4);
                    l2_prefetch(vals + r, 128 * sizeof(typename Fmt<DT>::V));
                }
            }
        }
#pragma unroll
        for (int i = 0; i < QPT; ++i)
            deposit(cur[i], q0 + (int64_t)i * TPB < nq ? 0xFu : 0u, !TAB_OBS2 || ((s * QPT + i) & 1) == 0);
    };
    int64_t s = 0;
    if (XB > 0) {
        // phases (block-uniform): block-synchronous / band mode until the
        // table streams in the uniform mode, then a loop with the uniform
        // deposit only (with the band mode compiled into the loop, one loop
        // for all modes costs the uniform mode ~4%; without it, the single
        // loop is the faster one)
        for (; s < steps && !tab.uniform(); ++s)  // block-uniform trip count
            step(s, [&](const QuadT<DT> &q, uint32_t in, bool obs) { tab.quad(q, in, flags, obs); });
        for (; s < steps; ++s)
            step(s, [&](const QuadT<DT> &q, uint32_t in, bool obs) { tab.fast_quad(q, in, flags, obs); });
    } else {
        for (; s < steps; ++s)
            step(s, [&](const QuadT<DT> &q, uint32_t in, bool obs) { tab.quad(q, in, flags, obs); });
    }
    // tail (< 4 rows, last block only)
    const int tail = (int)(row1 - row0 - 4 * nq);
    if (tail > 0) {  // block-uniform
        QuadT<DT> t;
        load_partial<DT>(keys, vals, row0 + 4 * nq, tid == 0 ? tail : 0, t);
        tab.quad(t, tid == 0 ? (1u << tail) - 1u : 0u, flags);
    }
    tab.finish();
#if TAB_DEBUG
    tab.dbg_flush(g_tab_modes);
#endif
    flags = __reduce_or_sync(0xffffffffu, flags);
    if ((tid & 31) == 0 && flags) atomicOr(status, flags);
}

template <int DT, int K, int TPB, int GQC, int XB>
int launch_table_t(const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t *kglob,
                   unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
    using Geo = TabGeom<DT, K, XB>;
    using V = typename Fmt<DT>::V;
    const size_t smem = GQC > 0 ? Geo::bytes_gqc(GQC) : Geo::bytes(G);
    if (GQC > 0 && Geo::gq(G) > GQC) return -1;
    if (smem > (size_t)device_props().smem_optin) return -1;
    const bool vec = (((uintptr_t)keys | (uintptr_t)vals) & 15) == 0;
    auto kern = vec ? k_table<DT, K, TPB, true, GQC, XB> : k_table<DT, K, TPB, false, GQC, XB>;
    static thread_local size_t configured[2] = {};
    if (configured[vec] < smem) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return -2;
        configured[vec] = smem;
    }
    if (n == 0) return 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TPB, smem);
    if (per_sm < 1) return -1;
    int64_t grid = (int64_t)per_sm * device_props().sms;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = (chunk + 3) & ~(int64_t)3;  // quad-aligned block ranges
    grid = (n + chunk - 1) / chunk;
    kern<<<(unsigned)grid, TPB, smem, st>>>(keys, (const V *)vals, n, G, chunk, kglob, slots, status);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace

int table_max_groups(int K, int DT) {
    const size_t cap = (size_t)device_props().smem_optin;
    const size_t per = 4 * (size_t)K * (DT == 1 ? 2 : 1) + 12;
    return (int)((cap - 64 - 1024) / per) - 8 - 32;  // (static shared memory comes out of the same budget; lane sinks)
}

int launch_table_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t *kglob,
                     unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
#define TAB_CASE(dt, k)                                                                                   \
    if (DT == dt && K == k)                                                                               \
        return G <= 1024 ? launch_table_t<dt, k, 256, 1056, 0>(keys, vals, n, G, kglob, slots, status, st, launches) \
             : G <= 2048 ? launch_table_t<dt, k, 256, 0, 0>(keys, vals, n, G, kglob, slots, status, st, launches)    \
             : TabGeom<dt, k, 1>::bytes(G) <= (size_t)device_props().smem_optin - 1024                              \
                         ? launch_table_t<dt, k, TAB_BIGTPB, 0, 1>(keys, vals, n, G, kglob, slots, status, st, launches)   \
                         : launch_table_t<dt, k, TAB_BIGTPB, 0, 0>(keys, vals, n, G, kglob, slots, status, st, launches);
    TAB_CASE(1, 1) TAB_CASE(1, 2) TAB_CASE(1, 3) TAB_CASE(1, 4)
    TAB_CASE(0, 1) TAB_CASE(0, 2) TAB_CASE(0, 3) TAB_CASE(0, 4)
#undef TAB_CASE
    return -1;
}

}  // namespace repro

#if TAB_DEBUG
// debug builds: calls per table mode of k_table since the last read (slow, band, uniform)
extern "C" int repro_debug_table_modes(unsigned long long *out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, repro::g_tab_modes, sizeof(unsigned long long) * 3);
    const unsigned long long z[3] = {0, 0, 0};
    cudaMemcpyToSymbol(repro::g_tab_modes, z, sizeof(z));
    return 0;
}
#endif
