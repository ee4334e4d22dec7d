// atoms_bench.cu -- shared-atomic throughput with precomputed addresses
// (16 unrolled ATOMS per iteration, no per-iteration address arithmetic).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define IT 2048
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }

template <int MODE>  // 0 random, 1 conflict-free (bank = lane), 2 same address per warp, 3 plain STS random, 4 LDS random
__global__ void k(uint32_t *out, int G) {
    extern __shared__ uint32_t t[];
    for (int i = threadIdx.x; i < G; i += blockDim.x) t[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t a[16];
    uint32_t s = hsh(blockIdx.x * 1024 + threadIdx.x);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        s = hsh(s + j);
        if (MODE == 0 || MODE == 3 || MODE == 4) a[j] = s % G;
        else if (MODE == 1) a[j] = ((s % (G / 32)) * 32 + lane);
        else a[j] = (hsh(blockIdx.x * 64 + (threadIdx.x >> 5) * 16 + j)) % G;
    }
    uint32_t acc = 0;
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (MODE == 3) t[a[j]] = i;
            else if (MODE == 4) acc += t[a[j] ^ (i & 1)];
            else atomicAdd(&t[a[j]], 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t[0] + acc;
}

template <int MODE>
void run(const char *name, int G, int tpb, int bps) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *o; cudaMalloc(&o, 4 * sms * bps);
    size_t smem = 4 * (size_t)G;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<MODE><<<sms * bps, tpb, smem>>>(o, G);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<sms * bps, tpb, smem>>>(o, G);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warp_ops = (double)sms * bps * (tpb / 32) * IT * 16;
    double clk = ms * 1e-3 * 1.965e9;  // nominal clock
    printf("%-34s G=%-6d %7.3f ms  %6.2f clk per warp-op per SM  (%5.2f lane-ops/clk/SM) %s\n", name, G, ms,
           clk / (warp_ops / sms), 32.0 * (warp_ops / sms) / clk, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<0>("ATOMS random", 1024, 256, 4);
    run<0>("ATOMS random", 8192, 256, 4);
    run<1>("ATOMS conflict-free", 8192, 256, 4);
    run<2>("ATOMS same address per warp", 8192, 256, 4);
    run<3>("STS random", 8192, 256, 4);
    run<4>("LDS random", 8192, 256, 4);
    run<1>("ATOMS conflict-free 512t", 8192, 512, 2);
    return 0;
}
