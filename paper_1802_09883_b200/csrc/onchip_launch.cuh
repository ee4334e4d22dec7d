// onchip_launch.cuh -- the on-chip GroupBy kernel template (one block per
// contiguous row range, accumulate_range of onchip_core.cuh) and its launcher,
// shared by the single-column path (k_onchip.cu) and the multi-column path
// (k_multi.cu).
#pragma once

#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"

#ifndef ONCHIP_TMA
#define ONCHIP_TMA 1
#endif

namespace repro {

int onchip_variant();  // k_onchip.cu: 0 auto, 1 atomic (TMA ring), 2 table, 3 atomic + register loads

template <int DT, int K, bool REGTOT, bool TMA, class SRC>
__global__ void __launch_bounds__(256, ONCHIP_MINBLOCKS)
k_onchip_accumulate(const int32_t *__restrict__ keys, const SRC src, int64_t n, int32_t G, int64_t chunk,
                    int32_t *__restrict__ kglob, unsigned long long *__restrict__ slots,
                    uint32_t *__restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int64_t row0 = (int64_t)blockIdx.x * chunk;
    const int64_t row1 = min(n, row0 + chunk);
    uint32_t flags = 0;
    PubArgs out{kglob, slots, nullptr, nullptr};
    accumulate_range<DT, K, REGTOT, 0, TMA, SRC>(keys, src, row0, row1, G, smem, flags, out);
    flags = __reduce_or_sync(0xffffffffu, flags);
    if ((threadIdx.x & 31) == 0 && flags) atomicOr(status, flags);
}

// Launch the on-chip kernel for row source SRC over Gv (virtual) groups.
// ALLOW_SMEM_SUMS instantiates the variant with level sums in shared memory
// (G > REG_GQ); the multi-column sources use register sums only.
template <int DT, int K, class SRC, bool ALLOW_SMEM_SUMS>
int launch_onchip_src(const int32_t *keys, const SRC &src, int64_t n, int32_t Gv, int32_t *kglob,
                      unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
    using Cfg = OnchipCfg<DT, K>;
    constexpr int TILE = Cfg::TPB * SRC::R;
    const bool regtot = Gv <= Cfg::REG_GQ;  // level sums in registers
    if (!regtot && !ALLOW_SMEM_SUMS) return -1;
    // TMA-fed ring when every column is 16-byte aligned and the ring fits
    uintptr_t align = (uintptr_t)keys;
    for (int j = 0; j < SRC::NCOL; ++j) align |= (uintptr_t)src.col[j];
    const size_t table = onchip_smem_bytes<DT, K>(Gv, regtot);
    const size_t ring = onchip_ring_bytes<DT, K, SRC::NCOL, SRC::R>();
    const bool tma = ONCHIP_TMA && onchip_variant() != 3 && (align & 15) == 0 &&
                     table + ring <= (size_t)device_props().smem_optin;
    void (*kern)(const int32_t *, const SRC, int64_t, int32_t, int64_t, int32_t *, unsigned long long *,
                 uint32_t *);
    if (regtot) {
        kern = tma ? k_onchip_accumulate<DT, K, true, true, SRC> : k_onchip_accumulate<DT, K, true, false, SRC>;
    } else {
        if constexpr (ALLOW_SMEM_SUMS)
            kern = tma ? k_onchip_accumulate<DT, K, false, true, SRC> : k_onchip_accumulate<DT, K, false, false, SRC>;
        else
            return -1;
    }
    const size_t smem = table + (tma ? ring : 0);
    if (smem > (size_t)device_props().smem_optin) return -1;
    static thread_local size_t configured[2][2] = {};
    if (configured[regtot][tma] < smem) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return -2;
        configured[regtot][tma] = smem;
    }
    if (n == 0) return 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::TPB, smem);
    if (per_sm < 1) return -1;
    int64_t grid = (int64_t)per_sm * device_props().sms;
    // a block's int64 level sums must not overflow: <= 2^23 rows per block
    const int64_t min_grid = (n + (1ll << 23) - 1) >> 23;
    if (grid < min_grid) grid = min_grid;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = ((chunk + TILE - 1) / TILE) * TILE;
    if (chunk > (1ll << 23)) chunk = (1ll << 23) / TILE * TILE;
    grid = (n + chunk - 1) / chunk;
    kern<<<(unsigned)grid, Cfg::TPB, smem, st>>>(keys, src, n, Gv, chunk, kglob, slots, status);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace repro
