// microbench.cu -- throughput of the primitives the on-chip accumulate kernel
// can be built from, on the whole GPU (148 SMs).  Prints operations per SM per
// cycle at the measured clock.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

// 32-bit shared atomicAdd on random slots of a G-entry table
__global__ void k_atoms(uint32_t *out, int G) {
    extern __shared__ uint32_t t[];
    for (int i = threadIdx.x; i < G; i += blockDim.x) t[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        atomicAdd(&t[(s >> 8) % G], s);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t[0];
}

// 32-bit shared atomicAdd with only every `G>>16`-th lane active (predicated)
__global__ void k_atoms_pred(uint32_t *out, int G) {
    extern __shared__ uint32_t t[];
    const int every = G >> 16, g = G & 0xFFFF;
    for (int i = threadIdx.x; i < g; i += blockDim.x) t[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    const bool on = (threadIdx.x % every) == 0;
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        if (on) atomicAdd(&t[(s >> 8) % g], s);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t[0];
}

// ATOMS with return value (histogram rank)
__global__ void k_atoms_ret(uint32_t *out, int G) {
    extern __shared__ uint32_t t[];
    for (int i = threadIdx.x; i < G; i += blockDim.x) t[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x), acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        acc += atomicAdd(&t[(s >> 8) % G], 1u);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// random STS.64 scatter + LDS.64 gather
__global__ void k_scatter(uint32_t *out, int G) {
    extern __shared__ unsigned long long b64[];
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    unsigned long long acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        b64[(s >> 8) % G] = s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G; i += blockDim.x) acc += b64[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)acc;
}

// 64-bit shared atomicAdd (CAS spin loop on sm_100a), random slots
__global__ void k_cas64(uint32_t *out, int G) {
    extern __shared__ unsigned long long c64[];
    for (int i = threadIdx.x; i < G; i += blockDim.x) c64[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        atomicAdd(&c64[(s >> 8) % G], (unsigned long long)s);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (uint32_t)c64[0];
}

// three 64-bit CAS adds per iteration into a [G][3] table (one row of fp64 K=3)
__global__ void k_cas64x3(uint32_t *out, int G) {
    extern __shared__ unsigned long long c3[];
    for (int i = threadIdx.x; i < 4 * G; i += blockDim.x) c3[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        unsigned long long *p = c3 + 4 * ((s >> 8) % G);
        atomicAdd(p, (unsigned long long)s);
        atomicAdd(p + 1, (unsigned long long)(s ^ 7));
        atomicAdd(p + 2, (unsigned long long)(s ^ 9));
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (uint32_t)c3[0];
}

// six 32-bit ATOMS per iteration into a [G][6] table (group-major layout)
__global__ void k_atoms6(uint32_t *out, int G) {
    extern __shared__ uint32_t a6[];
    for (int i = threadIdx.x; i < 6 * G; i += blockDim.x) a6[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        uint32_t *p = a6 + 6 * ((s >> 8) % G);
        atomicAdd(p, s); atomicAdd(p + 1, s ^ 1); atomicAdd(p + 2, s ^ 2);
        atomicAdd(p + 3, s ^ 3); atomicAdd(p + 4, s ^ 4); atomicAdd(p + 5, s ^ 5);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = a6[0];
}

// conflict-free ATOMS: lane l always hits bank l (random row of a [G/32][32] table)
__global__ void k_atoms_cf(uint32_t *out, int G) {
    extern __shared__ uint32_t tc[];
    for (int i = threadIdx.x; i < G; i += blockDim.x) tc[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, rows = G / 32;
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        atomicAdd(&tc[((s >> 8) % rows) * 32 + lane], s);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = tc[0];
}

// d-way bank conflicts: lanes l and l+32/d share a bank (different rows)
__global__ void k_atoms_dway(uint32_t *out, int G) {
    extern __shared__ uint32_t td[];
    const int d = G >> 16, g = G & 0xFFFF;
    for (int i = threadIdx.x; i < g; i += blockDim.x) td[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, rows = g / 32;
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        atomicAdd(&td[((s >> 8) % rows) * 32 + (lane % (32 / d))], s);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = td[0];
}

// plain 64-bit shared read-modify-write (warp-private region, no atomics)
__global__ void k_rmw64(uint32_t *out, int G) {
    extern __shared__ unsigned long long t64[];
    const int w = threadIdx.x >> 5;
    unsigned long long *my = t64 + w * G;
    for (int i = threadIdx.x & 31; i < G; i += 32) my[i] = 0;
    __syncwarp();
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        unsigned long long *p = &my[(s >> 8) % G];
        *p += s;
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = (uint32_t)my[0];
}

__global__ void k_match(uint32_t *out, int G) {
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x), acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        acc += __match_any_sync(0xffffffffu, (s >> 8) % G);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_redux(uint32_t *out, int G) {
    uint32_t s = hsh(blockIdx.x * blockDim.x + threadIdx.x), acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        s = s * 1664525u + 1013904223u;
        acc += __reduce_add_sync(0xffffffffu, s);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_dadd(uint32_t *out, int G) {
    double a = threadIdx.x, b = 1.0, c = 2.0, d = 3.0;
    const double e = 1.0000001;
    for (int i = 0; i < ITERS; ++i) {
        a = __dadd_rn(a, e); b = __dadd_rn(b, e); c = __dadd_rn(c, e); d = __dadd_rn(d, e);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)(a + b + c + d);
}

__global__ void k_f2i(uint32_t *out, int G) {
    double a = threadIdx.x * 1.5;
    long long acc = 0;
    for (int i = 0; i < ITERS; ++i) {
        acc += __double2ll_rn(a);
        a = __dadd_rn(a, 1.25);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)acc;
}

typedef void (*kfn)(uint32_t *, int);

static void run(const char *name, kfn k, int G, int tpb, int bps, size_t smem, double ops_per_thread_iter) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    uint32_t *out;
    cudaMalloc(&out, sizeof(uint32_t) * sms * bps * tpb);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = sms * bps;
    k<<<grid, tpb, smem>>>(out, G);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<grid, tpb, smem>>>(out, G);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    const double ops = 5.0 * grid * tpb * (double)ITERS * ops_per_thread_iter;
    const double per_sm_per_s = ops / (ms * 1e-3) / sms;
    printf("%-28s G=%-6d tpb=%-4d bps=%d  %8.3f ms  %10.3e op/s/SM  %6.2f op/clk/SM(@%.0fMHz nominal) %s\n", name, G,
           tpb, bps, ms, per_sm_per_s, per_sm_per_s / (clk_khz * 1e3), clk_khz / 1e3,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(out);
}

int main() {
    run("atoms conflict-free", k_atoms_cf, 4096, 256, 4, 4096 * 4, 1);
    run("atoms 2-way", k_atoms_dway, (2 << 16) | 4096, 256, 4, 4096 * 4, 1);
    run("atoms 4-way", k_atoms_dway, (4 << 16) | 4096, 256, 4, 4096 * 4, 1);
    run("atoms conflict-free 1024t", k_atoms_cf, 4096, 1024, 1, 4096 * 4, 1);
    for (int G : {1024, 4096}) {
        run("cas64 atomicAdd u64 random", k_cas64, G, 256, 4, G * 8, 1);
        run("cas64 x3 per row [G][4]", k_cas64x3, G, 256, 4, G * 32, 1);
        run("atoms x6 per row [G][6]", k_atoms6, G, 256, 4, G * 24, 1);
        run("cas64 x3 per row [G][4] 512t", k_cas64x3, G, 512, 2, G * 32, 1);
        run("atoms x6 per row [G][6] 512t", k_atoms6, G, 512, 2, G * 24, 1);
    }
    for (int G : {16, 1024, 4096}) {
        run("atoms.add.u32 random", k_atoms, G, 256, 4, G * 4, 1);
        run("atoms.add.u32 random", k_atoms, G, 1024, 1, G * 4, 1);
    }
    run("atoms.add.u32 G=1 (same addr)", k_atoms, 1, 256, 4, 4, 1);
    run("atoms 1/4 lanes active", k_atoms_pred, (4 << 16) | 1024, 256, 4, 1024 * 4, 0.25);
    run("atoms 1/8 lanes active", k_atoms_pred, (8 << 16) | 1024, 256, 4, 1024 * 4, 0.125);
    run("atoms 1/32 lanes active", k_atoms_pred, (32 << 16) | 1024, 256, 4, 1024 * 4, 1.0 / 32);
    run("atoms with return G=1024", k_atoms_ret, 1024, 256, 4, 1024 * 4, 1);
    run("sts.64 random scatter 4096", k_scatter, 4096, 256, 2, 4096 * 8, 1);
    for (int G : {64, 1024}) run("lds64+sts64 rmw warp-private", k_rmw64, G, 256, 1, (size_t)G * 8 * 8, 1);
    run("match.any G=1024", k_match, 1024, 256, 4, 0, 1);
    run("redux.sum", k_redux, 0, 256, 4, 0, 1);
    run("dadd (4 chains)", k_dadd, 0, 256, 4, 0, 4);
    run("f2i.s64.f64 + dadd", k_f2i, 0, 256, 4, 0, 1);
    return 0;
}
