// k_nvls.cu -- in-switch (NVLS) integer all-reduce of the absolute-level slot
// table for the multi-GPU exchange (the
// paper's setting for RSum is an MPI_Reduce across processes,
// PAPER.md:755-757).
//
// Every rank holds its table (status word, window tops kglob, slot words) at
// the same offsets of a symmetric buffer that is also mapped at a MULTICAST
// address (torch.distributed._symmetric_memory provides the mapping).  Rank r
// reduces the r-th slice of each region through the switch --
// multimem.ld_reduce (OR of the status bits, MAX of the tops, ADD of the
// slot words: all integer, so the result does not depend on the order the
// switch combines the ranks in) -- and writes the result back to every
// rank's copy with multimem.st.  The caller brackets the launch with
// symmetric-memory barriers (the deposits of every rank complete before, the
// stores of every rank visible after).
#include "common.cuh"
#include "internal.h"

#include <algorithm>

namespace repro {

namespace {

__device__ __forceinline__ uint32_t mm_or_b32(const uint32_t *p) {
    uint32_t v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void mm_st_b32(uint32_t *p, uint32_t v) {
    asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t mm_max_s32(const int32_t *p) {
    int32_t v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.max.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void mm_st_s32(int32_t *p, int32_t v) {
    asm volatile("multimem.st.relaxed.sys.global.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long mm_add_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void mm_st_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("multimem.st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// [lo, hi) of this rank's slice of n words
__device__ __forceinline__ void slice(int64_t n, int rank, int world, int64_t &lo, int64_t &hi) {
    const int64_t per = (n + world - 1) / world;
    lo = min(n, (int64_t)rank * per);
    hi = min(n, lo + per);
}

__global__ void __launch_bounds__(256)
k_nvls_reduce(uint32_t *mc_flags, int32_t *mc_kglob, int64_t nk, unsigned long long *mc_slots, int64_t ns, int rank,
              int world) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    if (t == 0 && rank == 0) mm_st_b32(mc_flags, mm_or_b32(mc_flags));
    int64_t lo, hi;
    slice(nk, rank, world, lo, hi);
    for (int64_t i = lo + t; i < hi; i += stride) mm_st_s32(mc_kglob + i, mm_max_s32(mc_kglob + i));
    slice(ns, rank, world, lo, hi);
    for (int64_t i = lo + t; i < hi; i += stride) mm_st_u64(mc_slots + i, mm_add_u64(mc_slots + i));
}

}  // namespace

int launch_nvls_reduce(uint32_t *mc_flags, int32_t *mc_kglob, int64_t nk, unsigned long long *mc_slots, int64_t ns,
                       int rank, int world, cudaStream_t st, int *launches) {
    const int64_t per = (ns + world - 1) / world;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * device_props().sms, (per + 255) / 256));
    k_nvls_reduce<<<grid, 256, 0, st>>>(mc_flags, mc_kglob, nk, mc_slots, ns, rank, world);
    ++*launches;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace repro
