// k_sparse.cu -- GroupBy-SUM over arbitrary int64 keys:
// the paper's operators hash their keys (HashAggregation);
// the dense path assumes identity hashing.  Here the keys are
// first mapped to dense group ids through a GPU hash table, then the dense
// reproducible GroupBy runs unchanged:
//   1. k_hash_insert   open addressing (linear probing, 64-bit CAS) of every
//                      row's key into a table of 2^b slots
//   2. k_hash_collect  the distinct keys (in table order)
//   3. sort            the distinct keys ascending (LSD radix sort of the
//                      64-bit slot words, 8 passes of 8-bit digits: k_rs_*):
//                      the dense id of a key is its rank, so ids -- and the
//                      output order -- depend only on the SET of keys
//   4. k_hash_assign   rank -> the key's slot
//   5. k_hash_map      every row's id
// The sums are the dense path's, so the result bits depend only on the
// multiset of (key, value) pairs.  Slots hold key ^ 2^63 (0 = empty, so the
// table is cleared with a memset); the key INT64_MIN is reserved (EKEY).
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace repro {

namespace {

constexpr unsigned long long FLIP = 0x8000000000000000ull;

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

// key -> table word: the key sign-extended to 64 bits with the top bit
// flipped (0 = empty slot, so INT64_MIN is reserved; no int32 key maps to 0)
template <typename KeyT>
__device__ __forceinline__ unsigned long long key_word(KeyT k) { return (unsigned long long)(int64_t)k ^ FLIP; }

template <typename KeyT>
__global__ void k_hash_insert(const KeyT *__restrict__ keys, int64_t n, unsigned long long *tk, uint64_t mask,
                              uint32_t *status, unsigned long long *distinct) {
    uint32_t bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long s = key_word(keys[i]);
        if (s == 0ull) {
            bad = FLAG_EKEY;
            continue;
        }
        uint64_t h = fmix64(s) & mask;
        // bounded probing: with more distinct keys than slots (the caller then
        // reports ENOMEM from the distinct count) a row gives up after a full turn
        for (uint64_t probe = 0; probe <= mask; ++probe) {
            const unsigned long long cur = tk[h];
            if (cur == s) break;
            if (cur == 0ull) {
                const unsigned long long prev = atomicCAS(&tk[h], 0ull, s);
                if (prev == 0ull) {
                    atomicAdd(distinct, 1ull);
                    break;
                }
                if (prev == s) break;
            }
            h = (h + 1) & mask;
        }
    }
    if (bad) atomicOr(status, bad);
}

__global__ void k_hash_collect(const unsigned long long *tk, uint64_t cap, unsigned long long *out,
                               unsigned long long *count) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long s = tk[i];
        if (s != 0ull) out[atomicAdd(count, 1ull)] = s;  // (slot word: unsigned order = key order)
    }
}

__device__ __forceinline__ uint64_t find_slot(const unsigned long long *tk, uint64_t mask, unsigned long long s) {
    uint64_t h = fmix64(s) & mask;
    while (tk[h] != s) h = (h + 1) & mask;  // every probed key is present
    return h;
}

__global__ void k_hash_assign(const unsigned long long *__restrict__ sorted, int64_t d, const unsigned long long *tk,
                              uint64_t mask, int32_t *tid, int64_t *keys_out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long s = sorted[i];
        tid[find_slot(tk, mask, s)] = (int32_t)i;
        keys_out[i] = (int64_t)(s ^ FLIP);
    }
}

// LSD radix sort of d distinct 64-bit words, 8-bit digits: per pass a tile
// histogram, then a stable scatter that derives its own offsets from all the
// tiles' histograms (digit base + the counts of the earlier tiles).  Tiles of
// RS_TILE words; the scatter ranks a tile in 8 rounds of 256 consecutive
// words (warp match -> rank among equal digits, per-warp counts -> prefix
// over the warps), so equal digits keep their order.
constexpr int RS_TPB = 256, RS_ROUNDS = 8, RS_TILE = RS_TPB * RS_ROUNDS;

__global__ void __launch_bounds__(RS_TPB)
k_rs_hist(const unsigned long long *__restrict__ in, int64_t d, int shift, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    const int tid = threadIdx.x;
    h[tid] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int i = tid; i < RS_TILE; i += RS_TPB)
        if (base + i < d) atomicAdd(&h[(unsigned)(in[base + i] >> shift) & 255u], 1u);
    __syncthreads();
    hist[(size_t)blockIdx.x * 256 + tid] = h[tid];  // tile-major
}

__global__ void __launch_bounds__(RS_TPB)
k_rs_scatter(const unsigned long long *__restrict__ in, unsigned long long *__restrict__ out, int64_t d, int shift,
             const uint32_t *__restrict__ hist, int nt) {
    __shared__ uint32_t wcnt[RS_TPB / 32][256];
    __shared__ uint32_t run[256];
    __shared__ uint32_t wsum[RS_TPB / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    unsigned long long x[RS_ROUNDS];  // the tile's words, loaded up front
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int64_t i = base + r * RS_TPB + tid;
        x[r] = i < d ? in[i] : 0ull;
    }
    {  // thread = digit: words of this digit in earlier tiles, and in all tiles
        uint32_t pre = 0, tot = 0;
#pragma unroll 8
        for (int t = 0; t < nt; ++t) {
            const uint32_t c = hist[(size_t)t * 256 + tid];
            pre += t < (int)blockIdx.x ? c : 0u;
            tot += c;
        }
        uint32_t incl = tot;  // exclusive scan of the digit totals over the block
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        uint32_t wb = 0;
        for (int w = 0; w < warp; ++w) wb += wsum[w];
        run[tid] = wb + incl - tot + pre;
    }
    for (int r = 0; r < RS_ROUNDS; ++r) {
#pragma unroll
        for (int w = 0; w < RS_TPB / 32; ++w) wcnt[w][tid] = 0;
        __syncthreads();
        const bool ok = base + r * RS_TPB + tid < d;
        const int dig = ok ? (int)((unsigned)(x[r] >> shift) & 255u) : 256;
        const unsigned peers = __match_any_sync(0xffffffffu, dig);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (ok && rank == 0) wcnt[warp][dig] = __popc(peers);
        __syncthreads();
        {  // thread = digit: exclusive prefix over the warps of this round
            uint32_t acc = run[tid];
#pragma unroll
            for (int w = 0; w < RS_TPB / 32; ++w) {
                const uint32_t c = wcnt[w][tid];
                wcnt[w][tid] = acc;
                acc += c;
            }
            run[tid] = acc;
        }
        __syncthreads();
        if (ok) out[wcnt[warp][dig] + rank] = x[r];
        __syncthreads();
    }
}

template <typename KeyT>
__global__ void k_hash_map(const KeyT *__restrict__ keys, int64_t n, const unsigned long long *tk, uint64_t mask,
                           const int32_t *__restrict__ tid, int32_t *ids) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long s = key_word(keys[i]);
        ids[i] = s == 0ull ? -1 : tid[find_slot(tk, mask, s)];
    }
}

int grid_for(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 16 * (int64_t)device_props().sms));
}

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

int rs_tiles(int64_t items) { return (int)((std::max<int64_t>(items, 1) + RS_TILE - 1) / RS_TILE); }

// radix sort scratch: the ping-pong buffer + the (tile, digit) counts
size_t sort_tmp_bytes(int64_t items) {
    return al256(8 * (size_t)std::max<int64_t>(items, 1)) + al256(4 * 256 * (size_t)rs_tiles(items));
}

}  // namespace

uint64_t sparse_table_slots(int64_t max_groups) {
    uint64_t cap = 1024;
    while (cap < 2 * (uint64_t)std::max<int64_t>(max_groups, 1)) cap <<= 1;
    return cap;
}

size_t sparse_scratch_bytes(int64_t n, int64_t max_groups) {
    const uint64_t cap = sparse_table_slots(max_groups);
    const size_t mg = (size_t)std::max<int64_t>(max_groups, 1);
    return al256(8 * cap) + al256(4 * cap) + al256(8 * mg) + al256(16) + al256(sort_tmp_bytes(max_groups)) +
           al256(4 * (size_t)std::max<int64_t>(n, 1));
}

// Map the keys to dense ids (ascending key order); `sorted_out` receives the
// distinct keys, *ids_out points at the int32 ids inside `scratch`, *d_out =
// number of distinct keys (the call synchronises `st` to read it).  Returns
// 0, -1 when there are more than max_groups distinct keys (*d_out still set),
// -2 on a CUDA error.
template <typename KeyT>
int sparse_map_keys(const KeyT *keys, int64_t n, int64_t max_groups, void *scratch, int64_t *sorted_out,
                    int32_t **ids_out, int64_t *d_out, uint32_t *status, cudaStream_t st, int *launches) {
    const uint64_t cap = sparse_table_slots(max_groups), mask = cap - 1;
    const size_t mg = (size_t)std::max<int64_t>(max_groups, 1);
    char *p = (char *)scratch;
    unsigned long long *tk = (unsigned long long *)p;
    p += al256(8 * cap);
    int32_t *tid = (int32_t *)p;
    p += al256(4 * cap);
    unsigned long long *dk = (unsigned long long *)p;  // distinct slot words (sorted in place)
    p += al256(8 * mg);
    unsigned long long *cnt = (unsigned long long *)p;  // [0] distinct (insert), [1] collected
    p += al256(16);
    const size_t tmp = sort_tmp_bytes(max_groups);
    void *ctmp = p;
    p += al256(tmp);
    int32_t *ids = (int32_t *)p;
    *ids_out = ids;
    if (cudaMemsetAsync(tk, 0, 8 * cap, st) != cudaSuccess || cudaMemsetAsync(cnt, 0, 16, st) != cudaSuccess)
        return -2;
    if (n > 0) {
        k_hash_insert<<<grid_for(n), 256, 0, st>>>(keys, n, tk, mask, status, cnt);
        ++*launches;
    }
    unsigned long long d = 0;
    if (cudaMemcpyAsync(&d, cnt, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
        return -2;
    *d_out = (int64_t)d;
    if ((int64_t)d > max_groups) return -1;
    if (d > 0) {
        k_hash_collect<<<grid_for((int64_t)cap), 256, 0, st>>>(tk, cap, dk, cnt + 1);
        ++*launches;
        (void)tmp;
        unsigned long long *alt = (unsigned long long *)ctmp;
        uint32_t *hist = (uint32_t *)((char *)ctmp + al256(8 * mg));
        const int nt = rs_tiles((int64_t)d);
        unsigned long long *src = dk, *dst = alt;
        for (int shift = 0; shift < 64; shift += 8) {  // 8 passes: the words end in dk
            k_rs_hist<<<nt, RS_TPB, 0, st>>>(src, (int64_t)d, shift, hist);
            k_rs_scatter<<<nt, RS_TPB, 0, st>>>(src, dst, (int64_t)d, shift, hist, nt);
            *launches += 2;
            std::swap(src, dst);
        }
        k_hash_assign<<<grid_for((int64_t)d), 256, 0, st>>>(dk, (int64_t)d, tk, mask, tid, sorted_out);
        ++*launches;
        k_hash_map<<<grid_for(n), 256, 0, st>>>(keys, n, tk, mask, tid, ids);
        ++*launches;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

template int sparse_map_keys<int64_t>(const int64_t *, int64_t, int64_t, void *, int64_t *, int32_t **, int64_t *,
                                      uint32_t *, cudaStream_t, int *);
template int sparse_map_keys<int32_t>(const int32_t *, int64_t, int64_t, void *, int64_t *, int32_t **, int64_t *,
                                      uint32_t *, cudaStream_t, int *);

}  // namespace repro
