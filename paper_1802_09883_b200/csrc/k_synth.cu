// k_synth.cu -- device-side copy of the seeded input generator of
// paper_1802_09883_b200/synth.py (bench / test support, NOT part of the
// method: it draws keys and values and holds none of the reproducible-sum
// arithmetic).  Counter-based SplitMix64 finaliser over (seed, column, row),
// multiply-shift range reduction; every value is an exactly representable
// integer divided once by 100.0 (correctly rounded), so the bits equal the
// numpy generator's -- tests/test_gpu_synth.py checks them on samples.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace repro {

namespace {

__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t col, uint64_t idx) {
    uint64_t z = seed ^ (col * 0xD6E8FEB86659FD93ull);
    z = z + (idx + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t uniform_int(uint64_t h, uint64_t R) { return ((h >> 32) * R) >> 32; }

// BASELINE config 4: keys U[0,G), qty 1+U{0..49}, price (90000+U{0..10410000})/100,
// disc U{0..10}/100, tax U{0..8}/100
__global__ void k_synth_q1(uint64_t seed, int64_t r0, int64_t n, int32_t G, int32_t *keys, double *qty,
                           double *price, double *disc, double *tax) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = (uint64_t)(r0 + i);
        keys[i] = (int32_t)uniform_int(splitmix(seed, 0, r), (uint64_t)G);
        qty[i] = 1.0 + (double)uniform_int(splitmix(seed, 1, r), 50);
        price[i] = __ddiv_rn(90000.0 + (double)uniform_int(splitmix(seed, 2, r), 10410001), 100.0);
        disc[i] = __ddiv_rn((double)uniform_int(splitmix(seed, 3, r), 11), 100.0);
        tax[i] = __ddiv_rn((double)uniform_int(splitmix(seed, 4, r), 9), 100.0);
    }
}

// BASELINE configs 0/1: keys U[0,G), values +-(1 + mant52 2^-52) 2^e, e U{-20..20}
__global__ void k_synth_mant_exp(uint64_t seed, int64_t r0, int64_t n, int32_t G, int32_t *keys, double *vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = (uint64_t)(r0 + i);
        keys[i] = (int32_t)uniform_int(splitmix(seed, 0, r), (uint64_t)G);
        const uint64_t h1 = splitmix(seed, 1, r), h2 = splitmix(seed, 2, r);
        const int64_t e = (int64_t)uniform_int(h2, 41) - 20;
        const uint64_t bits = ((h1 >> 63) << 63) | ((uint64_t)(e + 1023) << 52) | (h1 & ((1ull << 52) - 1));
        vals[i] = __longlong_as_double((long long)bits);
    }
}

// BASELINE config 2: keys U[0,G), values (h >> 11) 2^-52 - 1 in [-1, 1)
__global__ void k_synth_pm1(uint64_t seed, int64_t r0, int64_t n, int32_t G, int32_t *keys, double *vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = (uint64_t)(r0 + i);
        keys[i] = (int32_t)uniform_int(splitmix(seed, 0, r), (uint64_t)G);
        vals[i] = __dsub_rn(__dmul_rn((double)(splitmix(seed, 1, r) >> 11), 0x1p-52), 1.0);
    }
}

}  // namespace

int launch_synth(int config, uint64_t seed, int64_t r0, int64_t n, int32_t G, int32_t *keys, void *const *cols,
                 cudaStream_t st) {
    if (n <= 0) return 0;
    const int blocks = (int)((n + 255) / 256 < 16 * 148 ? (n + 255) / 256 : 16 * 148);
    if (config == 4)
        k_synth_q1<<<blocks, 256, 0, st>>>(seed, r0, n, G, keys, (double *)cols[0], (double *)cols[1],
                                           (double *)cols[2], (double *)cols[3]);
    else if (config == 0 || config == 1)
        k_synth_mant_exp<<<blocks, 256, 0, st>>>(seed, r0, n, G, keys, (double *)cols[0]);
    else if (config == 2)
        k_synth_pm1<<<blocks, 256, 0, st>>>(seed, r0, n, G, keys, (double *)cols[0]);
    else
        return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace repro
