// k_peak.cu -- measured FP add rate of this GPU: the FP side of SURVEY.md
// 8(d)'s roofline ("the slower of the input bytes over HBM and the deposit
// FLOPs at the vector FP64/FP32 peak").  The digit cascade costs 3K - 2
// correctly rounded adds per value (Alg. 1 lines 10-16, PAPER.md:666-672;
// per-level cost PAPER.md:881-889), so the FP roofline of a deposit is
// (3K - 2) * rows / rate.
//
// The kernel runs FP_CHAINS independent add chains per thread (enough to hide
// the pipe latency) on every SM, with a grid of a multiple of the SM count;
// the chains add a tiny constant to values near 1 so that every add is a
// normal, exactly specified _rn operation that the compiler cannot fold.
#include <cuda_runtime.h>

#include "internal.h"

namespace repro {

namespace {

constexpr int FP_CHAINS = 8;
constexpr int FP_ITERS = 4096;
constexpr int FP_TPB = 256;

template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }

template <typename T>
__global__ void __launch_bounds__(FP_TPB) k_fp_add_peak(T *out, T inc) {
    T a[FP_CHAINS];
#pragma unroll
    for (int c = 0; c < FP_CHAINS; ++c) a[c] = (T)1 + (T)(threadIdx.x * FP_CHAINS + c) * inc;
#pragma unroll 8
    for (int i = 0; i < FP_ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < FP_CHAINS; ++c) a[c] = add_rn(a[c], inc);
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < FP_CHAINS; ++c) s = add_rn(s, a[c]);
    if (s == (T)-1) out[blockIdx.x] = s;  // never true; keeps the chains live
}

}  // namespace

int measure_fp_add_rate(int DT, double *adds_per_s, cudaStream_t st) {
    const int sms = device_props().sms;
    const int blocks = sms * 8;
    void *scratch = nullptr;
    if (cudaMallocAsync(&scratch, (size_t)blocks * 8, st) != cudaSuccess) return -2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {  // rep 0 warms up; best of the other three
        cudaEventRecord(e0, st);
        if (DT == 1)
            k_fp_add_peak<double><<<blocks, FP_TPB, 0, st>>>((double *)scratch, 0x1p-40);
        else
            k_fp_add_peak<float><<<blocks, FP_TPB, 0, st>>>((float *)scratch, 0x1p-20f);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(scratch, st);
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) return -2;
    const double adds = (double)blocks * FP_TPB * FP_CHAINS * (FP_ITERS + 1);
    *adds_per_s = adds / (best * 1e-3);
    return 0;
}

}  // namespace repro
