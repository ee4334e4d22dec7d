// capi.cu -- host orchestration behind the C-ABI of include/repro_groupby.h:
// argument validation, path choice (on-chip tables vs radix partitioning),
// workspace layout, launches, device status word.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "repro_groupby.h"

namespace repro {

const DeviceProps &device_props() {
    static DeviceProps props[64];
    static bool have[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!have[dev]) {
        DeviceProps p{};
        p.device = dev;
        cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&p.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (p.sms <= 0) p.sms = 148;
        if (p.smem_optin <= 0) p.smem_optin = 227 * 1024;
        props[dev] = p;
        have[dev] = true;
    }
    return props[dev];
}

}  // namespace repro

using namespace repro;

namespace {

thread_local int32_t t_launches = 0;
thread_local int32_t t_path = -1;
int32_t g_path_override = -1;
// f3: group count up to which the
// on-chip path is used, per [dtype][fold] (0 = its capacity); see repro_autotune
int32_t g_onchip_cross[2][5] = {};

// ---- per-kernel event timing (repro_timing_enable / _collect) -------------
struct TimingRec {
    const char *name;
    cudaEvent_t a, b;
};
thread_local bool t_timing = false;
thread_local std::vector<TimingRec> t_recs;
thread_local std::vector<cudaEvent_t> t_pool;

cudaEvent_t pool_event() {
    if (!t_pool.empty()) {
        cudaEvent_t e = t_pool.back();
        t_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

thread_local std::vector<cudaEvent_t> t_open;

}  // namespace

namespace repro {
int trace_begin(cudaStream_t st) {
    if (!t_timing) return -1;
    cudaEvent_t a = pool_event();
    cudaEventRecord(a, st);
    t_open.push_back(a);
    return (int)t_open.size() - 1;
}
void trace_end(int token, const char *name, cudaStream_t st) {
    if (token < 0 || token >= (int)t_open.size()) return;
    cudaEvent_t b = pool_event();
    cudaEventRecord(b, st);
    t_recs.push_back({name, t_open[token], b});
    if (token == (int)t_open.size() - 1) t_open.pop_back();
}
}  // namespace repro

namespace {

// Run one launcher; when timing is on, bracket it with events on `st`.
template <class Fn>
int timed(const char *name, cudaStream_t st, Fn &&fn) {
    if (!t_timing) return fn();
    cudaEvent_t a = pool_event(), b = pool_event();
    cudaEventRecord(a, st);
    const int rc = fn();
    cudaEventRecord(b, st);
    t_recs.push_back({name, a, b});
    return rc;
}

constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

int status_from_flags(uint32_t f) {
    if (f & FLAG_ESTALL) return REPRO_ECUDA;
    if (f & FLAG_EINVAL) return REPRO_EINVAL;
    if (f & FLAG_EKEY) return REPRO_EKEY;
    if (f & FLAG_EDOM) return REPRO_EDOM;
    if (f & FLAG_ERANGE) return REPRO_ERANGE;
    return REPRO_OK;
}

int map_launch(int rc) { return rc == 0 ? REPRO_OK : (rc == -1 ? REPRO_EINVAL : REPRO_ECUDA); }

bool valid_shape(int32_t G, int32_t K, int32_t dt) {
    return G >= 1 && K >= 1 && K <= 4 && (dt == REPRO_F32 || dt == REPRO_F64);
}

// 0 = on-chip table, 1 = partitioned by the two-pass sweep (k_sweep.cu),
// 2 = partitioned by segmented radix passes (k_partition.cu: group counts
// beyond the sweep's 256 partitions), -1 = not supported
int choose_path(int32_t G, int32_t K, int32_t dt) {
    int onchip = onchip_max_groups(K, dt);
    const int32_t cross = g_onchip_cross[dt == REPRO_F64][K];
    if (cross > 0 && g_path_override < 0) onchip = std::min<int>(onchip, cross);
    const int part = G <= sweep_max_groups(K, dt) ? 1 : G <= partition_max_groups(K, dt) ? 2 : -1;
    if (g_path_override == 0) return G <= onchip ? 0 : -1;
    if (g_path_override == 1) return part;
    if (g_path_override == 2) return G <= partition_max_groups(K, dt) ? 2 : -1;
    if (G <= onchip) return 0;
    return part;
}

// on-chip workspace: [flags | kglob int32[G] | slots u64[G][NS][2]]
struct OnchipWs {
    uint32_t *flags;
    int32_t *kglob;
    unsigned long long *slots;
    size_t zero_bytes;  // bytes from flags to the end of slots (one memset)
};

size_t onchip_zero_bytes(int32_t G, int32_t K, int32_t dt) {
    return ALIGN + align_up(sizeof(int32_t) * (size_t)G) +
           align_up(sizeof(unsigned long long) * 2 * (size_t)G * slot_count(dt, K));
}

size_t onchip_ws_bytes(int64_t n, int32_t G, int32_t K, int32_t dt) {
    (void)n;
    return onchip_zero_bytes(G, K, dt);
}

OnchipWs carve_onchip(void *ws, int64_t n, int32_t G, int32_t K, int32_t dt) {
    OnchipWs w;
    char *p = (char *)ws;
    w.flags = (uint32_t *)p;
    w.kglob = (int32_t *)(p + ALIGN);
    w.slots = (unsigned long long *)(p + ALIGN + align_up(sizeof(int32_t) * (size_t)G));
    w.zero_bytes = onchip_zero_bytes(G, K, dt);
    (void)n;
    return w;
}

size_t ws_bytes_for(int path, int64_t n, int32_t G, int32_t K, int32_t dt) {
    if (path == 0) return onchip_ws_bytes(n, G, K, dt);
    if (path == 1) return ALIGN + sweep_workspace_bytes(n, G, K, dt);
    return ALIGN + partition_workspace_bytes(n, G, K, dt);
}

// Library-internal workspace cache for the blocking entry points.
struct Cache {
    std::mutex mu;
    void *ptr = nullptr;
    size_t bytes = 0;
    int device = -1;
} g_cache;

// Device buffers, streams and events of repro_groupby_sum_host, kept across
// calls (allocating ~0.2 GB and creating streams per call cost milliseconds).
struct HostCtx {
    static constexpr int NB = 3;
    std::mutex mu;
    int device = -1;
    cudaStream_t cs = nullptr, ks = nullptr;
    cudaEvent_t copied[NB] = {}, consumed[NB] = {};
    void *dbuf = nullptr, *dout = nullptr, *ws = nullptr, *pin = nullptr;
    size_t dbuf_b = 0, dout_b = 0, ws_b = 0, pin_b = 0;

    static int grow(void **p, size_t *have, size_t want, bool host) {
        if (*have >= want && *p) return REPRO_OK;
        if (*p) host ? cudaFreeHost(*p) : cudaFree(*p);
        *p = nullptr;
        *have = 0;
        if (want == 0) return REPRO_OK;
        if ((host ? cudaMallocHost(p, want) : cudaMalloc(p, want)) != cudaSuccess) {
            cudaGetLastError();
            *p = nullptr;
            return REPRO_ENOMEM;
        }
        *have = want;
        return REPRO_OK;
    }
    int prepare(size_t dbuf_want, size_t dout_want, size_t ws_want, size_t pin_want) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (device != dev) {  // (re)create per device; buffers of another device are dropped
            if (cs) cudaStreamDestroy(cs);
            if (ks) cudaStreamDestroy(ks);
            for (int b = 0; b < NB; ++b) {
                if (copied[b]) cudaEventDestroy(copied[b]);
                if (consumed[b]) cudaEventDestroy(consumed[b]);
            }
            dbuf = dout = ws = nullptr;
            dbuf_b = dout_b = ws_b = 0;
            if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess ||
                cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking) != cudaSuccess)
                return REPRO_ECUDA;
            for (int b = 0; b < NB; ++b)
                if (cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&consumed[b], cudaEventDisableTiming) != cudaSuccess)
                    return REPRO_ECUDA;
            device = dev;
        }
        int st = grow(&dbuf, &dbuf_b, dbuf_want, false);
        if (st == REPRO_OK) st = grow(&dout, &dout_b, std::max<size_t>(dout_want, 8), false);
        if (st == REPRO_OK) st = grow(&ws, &ws_b, std::max<size_t>(ws_want, ALIGN), false);
        if (st == REPRO_OK && pin_want) st = grow(&pin, &pin_b, pin_want, true);
        return st;
    }
    void release() {
        if (dbuf) cudaFree(dbuf);
        if (dout) cudaFree(dout);
        if (ws) cudaFree(ws);
        if (pin) cudaFreeHost(pin);
        dbuf = dout = ws = pin = nullptr;
        dbuf_b = dout_b = ws_b = pin_b = 0;
    }
} g_host;

void *cache_get(size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_cache.ptr && (g_cache.bytes < bytes || g_cache.device != dev)) {
        cudaFree(g_cache.ptr);
        g_cache.ptr = nullptr;
        g_cache.bytes = 0;
    }
    if (!g_cache.ptr) {
        size_t want = std::max(bytes, (size_t)1 << 20);
        if (cudaMalloc(&g_cache.ptr, want) != cudaSuccess) {
            cudaGetLastError();
            g_cache.ptr = nullptr;
            return nullptr;
        }
        g_cache.bytes = want;
        g_cache.device = dev;
    }
    return g_cache.ptr;
}

// Enqueue the whole GroupBy (deposit into a fresh slot table / partitions,
// then fold + Eq. 1 into out, or merge into an accumulator).  deposit_only:
// stop after the deposit (paths 0 and 1 leave the absolute-level slot table
// at the workspace's table offsets; the split form reads it from there).
int enqueue_groupby(const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t K, int32_t dt,
                    void *out, int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *ws,
                    size_t ws_bytes, cudaStream_t st, uint32_t **flags_out, bool deposit_only = false) {
    const int path = choose_path(G, K, dt);
    t_path = path;
    if (path < 0 || (deposit_only && path == 2)) return REPRO_EINVAL;
    if (ws_bytes < ws_bytes_for(path, n, G, K, dt)) return REPRO_ENOMEM;
    if (path == 0) {
        OnchipWs w = carve_onchip(ws, n, G, K, dt);
        *flags_out = w.flags;
        if (cudaMemsetAsync(ws, 0, w.zero_bytes, st) != cudaSuccess) return REPRO_ECUDA;
        const char *label = lean_single_applies(keys, vals, G) ? "lean_single"
                            : (onchip_variant() == 1 || onchip_variant() == 3) ? "onchip_accumulate"
                                                                                : "table_accumulate";
        int rc = timed(label, st, [&] {
            return launch_onchip_any(dt, K, keys, vals, n, G, w.kglob, w.slots, w.flags, st, &t_launches);
        });
        if (rc || deposit_only) return map_launch(rc);
        rc = timed("fold", st, [&] {
            return launch_fold(dt, K, G, w.kglob, w.slots, merge, acc_k, acc_C, acc_D, out, w.flags, st,
                               &t_launches);
        });
        return map_launch(rc);
    }
    uint32_t *flags = (uint32_t *)ws;
    *flags_out = flags;
    if (cudaMemsetAsync(flags, 0, ALIGN, st) != cudaSuccess) return REPRO_ECUDA;
    if (path == 1)
        return map_launch(launch_sweep(dt, K, keys, vals, n, G, (char *)ws + ALIGN, ws_bytes - ALIGN, merge,
                                       deposit_only ? nullptr : acc_k, acc_C, acc_D, deposit_only ? nullptr : out,
                                       flags, st, &t_launches));
    int rc = launch_partitioned(dt, K, keys, vals, n, G, (char *)ws + ALIGN, ws_bytes - ALIGN, merge, acc_k,
                                acc_C, acc_D, out, flags, st, &t_launches);
    return map_launch(rc);
}

int finish_blocking(uint32_t *d_flags, cudaStream_t st) {
    uint32_t f = 0;
    if (cudaMemcpyAsync(&f, d_flags, sizeof f, cudaMemcpyDeviceToHost, st) != cudaSuccess) return REPRO_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return REPRO_ECUDA;
    return status_from_flags(f);
}

}  // namespace

struct repro_acc {
    int32_t G, K, dt;
    int32_t *k;
    int64_t *C;
    int64_t *D;
};

extern "C" {

const char *repro_strerror(int status) {
    switch (status) {
        case REPRO_OK: return "ok";
        case REPRO_EINVAL: return "invalid argument";
        case REPRO_EKEY: return "key outside [0, n_groups)";
        case REPRO_EDOM: return "NaN or infinite value";
        case REPRO_ERANGE: return "value or carry count outside the representable range";
        case REPRO_ECUDA: return "CUDA error";
        case REPRO_ENOMEM: return "out of memory / workspace too small";
        default: return "unknown status";
    }
}

const char *repro_version(void) { return "repro_b200 0.1 (sm_100a)"; }

int32_t repro_last_launch_count(void) { return t_launches; }
int32_t repro_last_path(void) { return t_path; }
int32_t repro_onchip_max_groups(int32_t fold, int32_t dtype) {
    if (fold < 1 || fold > 4 || (dtype != 0 && dtype != 1)) return 0;
    return onchip_max_groups(fold, dtype);
}
int32_t repro_sweep_max_groups(int32_t fold, int32_t dtype) {
    if (fold < 1 || fold > 4 || (dtype != 0 && dtype != 1)) return 0;
    return sweep_max_groups(fold, dtype);
}
void repro_set_kernel_variant(int32_t variant) { set_onchip_variant(variant); }
void repro_set_route_mode(int32_t mode) { set_route_mode(mode); }

void repro_timing_enable(int32_t on) { t_timing = on != 0; }

int32_t repro_timing_collect(const char **names, int32_t *counts, double *total_ms, int32_t max) {
    std::vector<const char *> nm;
    std::vector<int32_t> cnt;
    std::vector<double> ms;
    for (auto &r : t_recs) {
        cudaEventSynchronize(r.b);
        float e = 0.f;
        cudaEventElapsedTime(&e, r.a, r.b);
        size_t i = 0;
        while (i < nm.size() && std::string(nm[i]) != r.name) ++i;
        if (i == nm.size()) {
            nm.push_back(r.name);
            cnt.push_back(0);
            ms.push_back(0.0);
        }
        cnt[i] += 1;
        ms[i] += e;
        t_pool.push_back(r.a);
        t_pool.push_back(r.b);
    }
    t_recs.clear();
    const int32_t k = (int32_t)std::min<size_t>(nm.size(), (size_t)std::max(max, 0));
    for (int32_t i = 0; i < k; ++i) {
        if (names) names[i] = nm[i];
        if (counts) counts[i] = cnt[i];
        if (total_ms) total_ms[i] = ms[i];
    }
    return k;
}

void repro_set_path_override(int32_t path) { g_path_override = (path >= 0 && path <= 2) ? path : -1; }

size_t repro_groupby_workspace_bytes(int64_t n, int32_t n_groups, int32_t fold, int32_t dtype) {
    if (n < 0 || !valid_shape(n_groups, fold, dtype)) return 0;
    const int path = choose_path(n_groups, fold, dtype);
    if (path < 0) return 0;
    return ws_bytes_for(path, n, n_groups, fold, dtype);
}

int repro_groupby_sum_async(const int32_t *keys, const void *vals, int64_t n, int32_t n_groups, int32_t fold,
                            int32_t dtype, void *out, void *workspace, size_t ws_bytes, void *stream,
                            int32_t *d_status) {
    t_launches = 0;
    if (n < 0 || !valid_shape(n_groups, fold, dtype) || !out || !workspace || !d_status) return REPRO_EINVAL;
    if (n > 0 && (!keys || !vals)) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *flags = nullptr;
    int rc = enqueue_groupby(keys, vals, n, n_groups, fold, dtype, out, 0, nullptr, nullptr, nullptr, workspace,
                             ws_bytes, st, &flags);
    if (rc != REPRO_OK) return rc;
    return map_launch(timed("status", st, [&] { return launch_status(flags, d_status, st, &t_launches); }));
}

int repro_groupby_sum(const int32_t *keys, const void *vals, int64_t n, int32_t n_groups, int32_t fold,
                      int32_t dtype, void *out) {
    t_launches = 0;
    if (n < 0 || !valid_shape(n_groups, fold, dtype) || !out) return REPRO_EINVAL;
    if (n > 0 && (!keys || !vals)) return REPRO_EINVAL;
    const size_t need = repro_groupby_workspace_bytes(n, n_groups, fold, dtype);
    if (need == 0) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    void *ws = cache_get(need);
    if (!ws) return REPRO_ENOMEM;
    uint32_t *flags = nullptr;
    int rc = enqueue_groupby(keys, vals, n, n_groups, fold, dtype, out, 0, nullptr, nullptr, nullptr, ws, need,
                             0, &flags);
    if (rc != REPRO_OK) {
        cudaStreamSynchronize(0);
        return rc;
    }
    return finish_blocking(flags, 0);
}

// ---- split form of the single-column GroupBy (multi-GPU exchange) ---------

int repro_groupby_table(int64_t n, int32_t n_groups, int32_t fold, int32_t dtype, int64_t *offsets,
                        int64_t *counts) {
    if (n < 0 || !valid_shape(n_groups, fold, dtype) || !offsets || !counts) return REPRO_EINVAL;
    const int path = choose_path(n_groups, fold, dtype);
    if (path != 0 && path != 1) return REPRO_EINVAL;
    OnchipWs w = carve_onchip(nullptr, n, n_groups, fold, dtype);  // path 1 uses the same leading layout
    offsets[0] = (int64_t)(uintptr_t)w.flags;
    offsets[1] = (int64_t)(uintptr_t)w.kglob;
    offsets[2] = (int64_t)(uintptr_t)w.slots;
    counts[0] = 1;
    counts[1] = n_groups;
    counts[2] = (int64_t)n_groups * slot_count(dtype, fold) * 2;
    return REPRO_OK;
}

int repro_nvls_table_allreduce_async(void *mc_workspace, const int64_t *offsets, const int64_t *counts, int32_t rank,
                                     int32_t world, void *stream) {
    t_launches = 0;
    if (!mc_workspace || !offsets || !counts || world < 1 || rank < 0 || rank >= world) return REPRO_EINVAL;
    if (((uintptr_t)mc_workspace) % ALIGN || offsets[0] % 4 || offsets[1] % 4 || offsets[2] % 8 || counts[0] != 1)
        return REPRO_EINVAL;
    char *b = (char *)mc_workspace;
    cudaStream_t st = (cudaStream_t)stream;
    return map_launch(timed("nvls_reduce", st, [&] {
        return launch_nvls_reduce((uint32_t *)(b + offsets[0]), (int32_t *)(b + offsets[1]), counts[1],
                                  (unsigned long long *)(b + offsets[2]), counts[2], rank, world, st, &t_launches);
    }));
}

int repro_groupby_deposit_async(const int32_t *keys, const void *vals, int64_t n, int32_t n_groups, int32_t fold,
                                int32_t dtype, void *workspace, size_t ws_bytes, void *stream) {
    t_launches = 0;
    if (n < 0 || !valid_shape(n_groups, fold, dtype) || !workspace) return REPRO_EINVAL;
    if (n > 0 && (!keys || !vals)) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    uint32_t *flags = nullptr;
    return enqueue_groupby(keys, vals, n, n_groups, fold, dtype, nullptr, 0, nullptr, nullptr, nullptr, workspace,
                           ws_bytes, (cudaStream_t)stream, &flags, true);
}

int repro_groupby_finish_async(int64_t n, int32_t n_groups, int32_t fold, int32_t dtype, void *out, void *workspace,
                               size_t ws_bytes, void *stream, int32_t *d_status) {
    t_launches = 0;
    if (n < 0 || !valid_shape(n_groups, fold, dtype) || !out || !workspace || !d_status) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    const int path = choose_path(n_groups, fold, dtype);
    if ((path != 0 && path != 1) || ws_bytes < ws_bytes_for(path, n, n_groups, fold, dtype)) return REPRO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    OnchipWs w = carve_onchip(workspace, n, n_groups, fold, dtype);
    int rc = timed("fold", st, [&] {
        return launch_fold(dtype, fold, n_groups, w.kglob, w.slots, 0, nullptr, nullptr, nullptr, out, w.flags, st,
                           &t_launches);
    });
    if (rc) return map_launch(rc);
    return map_launch(timed("status", st, [&] { return launch_status(w.flags, d_status, st, &t_launches); }));
}

int repro_groupby_window_limbs_async(int64_t n, int32_t n_groups, int32_t fold, int32_t dtype,
                                     const int32_t *k_global, int64_t *limbs, void *workspace, size_t ws_bytes,
                                     void *stream) {
    t_launches = 0;
    if (n < 0 || !valid_shape(n_groups, fold, dtype) || !k_global || !limbs || !workspace) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    const int path = choose_path(n_groups, fold, dtype);
    if ((path != 0 && path != 1) || ws_bytes < ws_bytes_for(path, n, n_groups, fold, dtype)) return REPRO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    OnchipWs w = carve_onchip(workspace, n, n_groups, fold, dtype);
    return map_launch(timed("slot_limbs", st, [&] {
        return launch_slot_limbs(dtype, fold, n_groups, k_global, w.slots, limbs, st, &t_launches);
    }));
}

int repro_groupby_finish_limbs_async(int64_t n, int32_t n_groups, int32_t fold, int32_t dtype, int32_t g0,
                                     int32_t count, const int32_t *k_range, const int64_t *limbs_range,
                                     void *out_range, void *workspace, size_t ws_bytes, void *stream,
                                     int32_t *d_status) {
    t_launches = 0;
    if (n < 0 || !valid_shape(n_groups, fold, dtype) || !workspace || !d_status) return REPRO_EINVAL;
    if (g0 < 0 || count < 0 || (int64_t)g0 + count > n_groups) return REPRO_EINVAL;
    if (count > 0 && (!k_range || !limbs_range || !out_range)) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    const int path = choose_path(n_groups, fold, dtype);
    if ((path != 0 && path != 1) || ws_bytes < ws_bytes_for(path, n, n_groups, fold, dtype)) return REPRO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    OnchipWs w = carve_onchip(workspace, n, n_groups, fold, dtype);
    int rc = timed("limbs_finalize", st, [&] {
        return launch_limbs_finalize(dtype, fold, count, k_range, limbs_range, out_range, w.flags, st, &t_launches);
    });
    if (rc) return map_launch(rc);
    return map_launch(timed("status", st, [&] { return launch_status(w.flags, d_status, st, &t_launches); }));
}

// ---- multi-column GroupBy (several SUMs + COUNT in one pass) ---------------

}  // extern "C"

namespace {

int multi_nout(int32_t proj, int32_t ncols) { return proj == 1 ? 4 : proj == 2 ? 2 : ncols; }

bool multi_valid(int64_t n, int32_t G, int32_t ncols, int32_t proj, int32_t K, int32_t dt) {
    if (n < 0 || !valid_shape(G, K, dt)) return false;
    if (proj == 1) return ncols == 4 && dt == REPRO_F64;
    if (proj == 2) return ncols == 1;
    return proj == 0 && ncols >= 1 && ncols <= 8;
}

// fused on-chip kernel applies: virtual groups G * NV fit the register tables
bool multi_fused(int32_t G, int32_t ncols, int32_t proj) {
    const int nv = multi_virtual_columns(proj, ncols);
    return nv > 0 && (int64_t)G * nv <= 1024;
}

// fused workspace: [on-chip zeroed region for G*NV groups | virtual results]
// fallback workspace: [flags accumulator | 2 projected columns (proj 1) |
// one single-column workspace, reused column after column]
size_t multi_ws_bytes(int64_t n, int32_t G, int32_t ncols, int32_t proj, int32_t K, int32_t dt) {
    const size_t vsz = dt == REPRO_F64 ? 8 : 4;
    if (multi_fused(G, ncols, proj)) {
        const int32_t Gv = G * multi_virtual_columns(proj, ncols);
        return onchip_ws_bytes(n, Gv, K, dt) + align_up(vsz * (size_t)Gv);
    }
    const int path = choose_path(G, K, dt);
    if (path < 0) return 0;
    const size_t vsz_ = dt == REPRO_F64 ? 8 : 4;
    const size_t proj_bytes = proj == 1 ? 2 * align_up(8 * (size_t)n) : proj == 2 ? align_up(vsz_ * (size_t)n) : 0;
    return ALIGN + proj_bytes + ws_bytes_for(path, n, G, K, dt);
}

// phase: 3 = whole call; 1 = zero + deposit only (multi-GPU split form);
// 2 = fold + scatter only (after the slot tables were all-reduced)
int enqueue_multi(const int32_t *keys, const void *const *cols, int32_t ncols, int32_t proj, int64_t n, int32_t G,
                  int32_t K, int32_t dt, void *const *outs, int64_t *counts, void *ws, size_t ws_bytes,
                  cudaStream_t st, uint32_t **flags_out, int phase = 3) {
    if (ws_bytes < multi_ws_bytes(n, G, ncols, proj, K, dt)) return REPRO_ENOMEM;
    const int nout = multi_nout(proj, ncols);
    if (multi_fused(G, ncols, proj)) {
        const int nv = multi_virtual_columns(proj, ncols);
        const int32_t Gv = G * nv;
        t_path = 2;
        OnchipWs w = carve_onchip(ws, n, Gv, K, dt);
        void *vout = (char *)ws + onchip_ws_bytes(n, Gv, K, dt);
        *flags_out = w.flags;
        if (phase & 1) {
            if (cudaMemsetAsync(ws, 0, w.zero_bytes, st) != cudaSuccess) return REPRO_ECUDA;
            const char *label = lean_multi_applies(dt, proj, ncols, keys, cols, G) ? "lean_multi" : "onchip_accumulate";
            int rc = timed(label, st, [&] {
                return launch_onchip_multi(dt, K, proj, ncols, keys, cols, n, G, w.kglob, w.slots, w.flags, st,
                                           &t_launches);
            });
            if (rc) return map_launch(rc);
        }
        if (!(phase & 2)) return REPRO_OK;
        int rc = timed("fold", st, [&] {
            return launch_fold(dt, K, Gv, w.kglob, w.slots, 0, nullptr, nullptr, nullptr, vout, w.flags, st,
                               &t_launches);
        });
        if (rc) return map_launch(rc);
        rc = timed("scatter", st, [&] {
            return launch_multi_scatter(dt, K, vout, G, nout, outs, w.slots, counts, st, &t_launches);
        });
        return map_launch(rc);
    }
    // fallback: one GroupBy pass per output column (projection materialised),
    // COUNT by integer atomics; status bits OR-ed over the passes
    t_path = 3;
    char *p = (char *)ws;
    uint32_t *acc = (uint32_t *)p;
    p += ALIGN;
    *flags_out = acc;
    if (cudaMemsetAsync(acc, 0, ALIGN, st) != cudaSuccess) return REPRO_ECUDA;
    const void *src[4] = {nullptr, nullptr, nullptr, nullptr};
    if (proj == 1) {
        double *dp = (double *)p, *charge = (double *)(p + align_up(8 * (size_t)n));
        p += 2 * align_up(8 * (size_t)n);
        int rc = timed("project", st, [&] {
            return launch_q1_project((const double *)cols[1], (const double *)cols[2], (const double *)cols[3], n,
                                     dp, charge, st, &t_launches);
        });
        if (rc) return map_launch(rc);
        src[0] = cols[0];
        src[1] = cols[1];
        src[2] = dp;
        src[3] = charge;
    } else if (proj == 2) {
        void *sq = p;
        p += align_up((dt == REPRO_F64 ? 8 : 4) * (size_t)n);
        int rc = timed("project", st, [&] { return launch_square(dt, cols[0], n, sq, st, &t_launches); });
        if (rc) return map_launch(rc);
        src[0] = cols[0];
        src[1] = sq;
    }
    const size_t rest = ws_bytes - (size_t)(p - (char *)ws);
    for (int c = 0; c < nout; ++c) {
        uint32_t *f = nullptr;
        int rc = enqueue_groupby(keys, proj != 0 ? src[c] : cols[c], n, G, K, dt, outs[c], 0, nullptr, nullptr,
                                 nullptr, p, rest, st, &f);
        if (rc != REPRO_OK) return rc;
        rc = launch_flags_or(acc, f, st, &t_launches);
        if (rc) return map_launch(rc);
    }
    if (counts) {
        int rc = timed("count", st, [&] { return launch_count_rows(keys, n, G, counts, st, &t_launches); });
        if (rc) return map_launch(rc);
    }
    t_path = 3;
    return REPRO_OK;
}

bool multi_ptrs_ok(int64_t n, const int32_t *keys, const void *const *cols, int32_t ncols, void *const *outs,
                   int nout) {
    if (!cols || !outs) return false;
    for (int c = 0; c < nout; ++c)
        if (!outs[c]) return false;
    if (n > 0) {
        if (!keys) return false;
        for (int c = 0; c < ncols; ++c)
            if (!cols[c]) return false;
    }
    return true;
}

}  // namespace

extern "C" {

int repro_groupby_multi_table(int64_t n, int32_t n_groups, int32_t ncols, int32_t proj, int32_t fold,
                              int32_t dtype, int64_t *offsets, int64_t *counts) {
    if (!multi_valid(n, n_groups, ncols, proj, fold, dtype) || !offsets || !counts) return REPRO_EINVAL;
    if (!multi_fused(n_groups, ncols, proj)) return REPRO_EINVAL;
    const int32_t Gv = n_groups * multi_virtual_columns(proj, ncols);
    OnchipWs w = carve_onchip(nullptr, n, Gv, fold, dtype);
    offsets[0] = (int64_t)(uintptr_t)w.flags;
    offsets[1] = (int64_t)(uintptr_t)w.kglob;
    offsets[2] = (int64_t)(uintptr_t)w.slots;
    counts[0] = 1;
    counts[1] = Gv;
    counts[2] = (int64_t)Gv * slot_count(dtype, fold) * 2;
    return REPRO_OK;
}

int repro_groupby_multi_deposit_async(const int32_t *keys, const void *const *cols, int32_t ncols, int32_t proj,
                                      int64_t n, int32_t n_groups, int32_t fold, int32_t dtype, void *workspace,
                                      size_t ws_bytes, void *stream) {
    t_launches = 0;
    if (!multi_valid(n, n_groups, ncols, proj, fold, dtype) || !workspace) return REPRO_EINVAL;
    if (!multi_fused(n_groups, ncols, proj)) return REPRO_EINVAL;
    if (n > 0 && (!keys || !cols)) return REPRO_EINVAL;
    for (int c = 0; c < ncols && n > 0; ++c)
        if (!cols[c]) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    uint32_t *flags = nullptr;
    return enqueue_multi(keys, cols, ncols, proj, n, n_groups, fold, dtype, nullptr, nullptr, workspace, ws_bytes,
                         (cudaStream_t)stream, &flags, 1);
}

int repro_groupby_multi_finish_async(int64_t n, int32_t n_groups, int32_t ncols, int32_t proj, int32_t fold,
                                     int32_t dtype, void *const *outs, int64_t *counts, void *workspace,
                                     size_t ws_bytes, void *stream, int32_t *d_status) {
    t_launches = 0;
    if (!multi_valid(n, n_groups, ncols, proj, fold, dtype) || !workspace || !d_status) return REPRO_EINVAL;
    if (!multi_fused(n_groups, ncols, proj)) return REPRO_EINVAL;
    const int nout = multi_nout(proj, ncols);
    if (!outs) return REPRO_EINVAL;
    for (int c = 0; c < nout; ++c)
        if (!outs[c]) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *flags = nullptr;
    int rc = enqueue_multi(nullptr, nullptr, ncols, proj, n, n_groups, fold, dtype, outs, counts, workspace, ws_bytes,
                           st, &flags, 2);
    if (rc != REPRO_OK) return rc;
    return map_launch(timed("status", st, [&] { return launch_status(flags, d_status, st, &t_launches); }));
}

size_t repro_groupby_multi_workspace_bytes(int64_t n, int32_t n_groups, int32_t ncols, int32_t proj, int32_t fold,
                                           int32_t dtype) {
    if (!multi_valid(n, n_groups, ncols, proj, fold, dtype)) return 0;
    return multi_ws_bytes(n, n_groups, ncols, proj, fold, dtype);
}

int repro_groupby_sum_multi_async(const int32_t *keys, const void *const *cols, int32_t ncols, int32_t proj,
                                  int64_t n, int32_t n_groups, int32_t fold, int32_t dtype, void *const *outs,
                                  int64_t *counts, void *workspace, size_t ws_bytes, void *stream,
                                  int32_t *d_status) {
    t_launches = 0;
    if (!multi_valid(n, n_groups, ncols, proj, fold, dtype) || !workspace || !d_status) return REPRO_EINVAL;
    if (!multi_ptrs_ok(n, keys, cols, ncols, outs, multi_nout(proj, ncols))) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *flags = nullptr;
    int rc = enqueue_multi(keys, cols, ncols, proj, n, n_groups, fold, dtype, outs, counts, workspace, ws_bytes, st,
                           &flags);
    if (rc != REPRO_OK) return rc;
    return map_launch(timed("status", st, [&] { return launch_status(flags, d_status, st, &t_launches); }));
}

int repro_groupby_sum_multi(const int32_t *keys, const void *const *cols, int32_t ncols, int32_t proj, int64_t n,
                            int32_t n_groups, int32_t fold, int32_t dtype, void *const *outs, int64_t *counts) {
    t_launches = 0;
    if (!multi_valid(n, n_groups, ncols, proj, fold, dtype)) return REPRO_EINVAL;
    if (!multi_ptrs_ok(n, keys, cols, ncols, outs, multi_nout(proj, ncols))) return REPRO_EINVAL;
    const size_t need = multi_ws_bytes(n, n_groups, ncols, proj, fold, dtype);
    if (need == 0) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    void *ws = cache_get(need);
    if (!ws) return REPRO_ENOMEM;
    uint32_t *flags = nullptr;
    int rc = enqueue_multi(keys, cols, ncols, proj, n, n_groups, fold, dtype, outs, counts, ws, need, 0, &flags);
    if (rc != REPRO_OK) {
        cudaStreamSynchronize(0);
        return rc;
    }
    return finish_blocking(flags, 0);
}

int repro_synth_generate(int32_t config, uint64_t seed, int64_t r0, int64_t n, int32_t n_groups, int32_t *keys,
                         void *const *cols, void *stream) {
    if (n < 0 || n_groups < 1 || (n > 0 && (!keys || !cols))) return REPRO_EINVAL;
    const int ncol = config == 4 ? 4 : 1;
    for (int c = 0; c < ncol && n > 0; ++c)
        if (!cols[c]) return REPRO_EINVAL;
    const int rc = launch_synth(config, seed, r0, n, n_groups, keys, cols, (cudaStream_t)stream);
    return rc == -1 ? REPRO_EINVAL : map_launch(rc);
}

int repro_measure_fp_add_rate(int32_t dtype, double *adds_per_s, void *stream) {
    if ((dtype != 0 && dtype != 1) || !adds_per_s) return REPRO_EINVAL;
    return map_launch(measure_fp_add_rate(dtype, adds_per_s, (cudaStream_t)stream));
}

}  // extern "C"

namespace {
template <typename KeyT>
int groupby_sum_sparse_impl(const KeyT *keys, const void *vals, int64_t n, int64_t max_groups, int32_t fold,
                            int32_t dtype, int64_t *out_keys, void *out_vals, int64_t *n_groups_out) {
    t_launches = 0;
    if (n < 0 || max_groups < 1 || max_groups > partition_max_groups(fold, dtype) || !valid_shape(1, fold, dtype) ||
        !out_keys || !out_vals || !n_groups_out)
        return REPRO_EINVAL;
    if (n > 0 && (!keys || !vals)) return REPRO_EINVAL;
    *n_groups_out = 0;
    const int32_t gmax = (int32_t)max_groups;
    const int pmax = choose_path(gmax, fold, dtype);
    if (pmax < 0) return REPRO_EINVAL;
    const int32_t gon = std::min<int32_t>(gmax, onchip_max_groups(fold, dtype));
    const size_t dense = std::max(ws_bytes_for(pmax, n, gmax, fold, dtype), ws_bytes_for(0, n, gon, fold, dtype));
    const size_t sp = align_up(sparse_scratch_bytes(n, max_groups));
    std::lock_guard<std::mutex> lock(g_cache.mu);
    void *ws = cache_get(ALIGN + sp + dense);
    if (!ws) return REPRO_ENOMEM;
    uint32_t *mflags = (uint32_t *)ws;
    if (cudaMemsetAsync(mflags, 0, 4, 0) != cudaSuccess) return REPRO_ECUDA;
    int32_t *ids = nullptr;
    int64_t d = 0;
    int rc = sparse_map_keys(keys, n, max_groups, (char *)ws + ALIGN, out_keys, &ids, &d, mflags, 0, &t_launches);
    *n_groups_out = d;
    if (rc == -1) return REPRO_ENOMEM;
    if (rc) return REPRO_ECUDA;
    uint32_t f = 0;
    if (cudaMemcpy(&f, mflags, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return REPRO_ECUDA;
    if (f) return status_from_flags(f);
    if (d == 0) return REPRO_OK;
    uint32_t *flags = nullptr;
    rc = enqueue_groupby(ids, vals, n, (int32_t)d, fold, dtype, out_vals, 0, nullptr, nullptr, nullptr,
                         (char *)ws + ALIGN + sp, dense, 0, &flags);
    if (rc != REPRO_OK) {
        cudaStreamSynchronize(0);
        return rc;
    }
    return finish_blocking(flags, 0);
}
}  // namespace

extern "C" {

int repro_groupby_sum_sparse(const int64_t *keys, const void *vals, int64_t n, int64_t max_groups, int32_t fold,
                             int32_t dtype, int64_t *out_keys, void *out_vals, int64_t *n_groups_out) {
    return groupby_sum_sparse_impl(keys, vals, n, max_groups, fold, dtype, out_keys, out_vals, n_groups_out);
}

int repro_groupby_sum_sparse_i32(const int32_t *keys, const void *vals, int64_t n, int64_t max_groups, int32_t fold,
                                 int32_t dtype, int64_t *out_keys, void *out_vals, int64_t *n_groups_out) {
    return groupby_sum_sparse_impl(keys, vals, n, max_groups, fold, dtype, out_keys, out_vals, n_groups_out);
}

int repro_groupby_moments(const int32_t *keys, const void *vals, int64_t n, int32_t n_groups, int32_t fold,
                          int32_t dtype, void *sum, void *avg, void *var, void *stddev, int64_t *counts) {
    t_launches = 0;
    if (!multi_valid(n, n_groups, 1, 2, fold, dtype) || !sum || !counts) return REPRO_EINVAL;
    if (n > 0 && (!keys || !vals)) return REPRO_EINVAL;
    const size_t vsz = dtype == REPRO_F64 ? 8 : 4;
    const size_t need = multi_ws_bytes(n, n_groups, 1, 2, fold, dtype);
    if (need == 0) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    void *ws = cache_get(need + align_up(vsz * (size_t)n_groups));
    if (!ws) return REPRO_ENOMEM;
    void *sumsq = (char *)ws + need;  // SUM(x^2) lives after the multi workspace
    void *outs[2] = {sum, sumsq};
    const void *cols[1] = {vals};
    uint32_t *flags = nullptr;
    int rc = enqueue_multi(keys, cols, 1, 2, n, n_groups, fold, dtype, outs, counts, ws, need, 0, &flags);
    if (rc == REPRO_OK)
        rc = map_launch(timed("moments", 0, [&] {
            return launch_moments(dtype, sum, sumsq, counts, n_groups, avg, var, stddev, 0, &t_launches);
        }));
    if (rc != REPRO_OK) {
        cudaStreamSynchronize(0);
        return rc;
    }
    return finish_blocking(flags, 0);
}

// ---- keyless single-array SUM / dot product (f4) ----------------------------

size_t repro_dot_workspace_bytes(int32_t fold, int32_t dtype) {
    return valid_shape(1, fold, dtype) ? onchip_ws_bytes(0, 1, fold, dtype) : 0;
}

}  // extern "C"

namespace {

// phase: 3 = whole call; 1 = zero + deposit (multi-GPU split form); 2 = fold
// + Eq. 1 only (after the slot tables were all-reduced)
int enqueue_array(const void *x, const void *y, int64_t n, int32_t K, int32_t dt, void *out, void *ws,
                  cudaStream_t st, uint32_t **flags_out, int phase = 3) {
    OnchipWs w = carve_onchip(ws, n, 1, K, dt);
    *flags_out = w.flags;
    t_path = 0;
    if (phase & 1) {
        if (cudaMemsetAsync(ws, 0, w.zero_bytes, st) != cudaSuccess) return REPRO_ECUDA;
        // register-state kernel (k_array.cu) for 16-byte aligned arrays; the
        // keyless on-chip kernel otherwise (or when a kernel variant is forced)
        const bool aligned = (((uintptr_t)x | (uintptr_t)y) & 15) == 0;
        int rc = (aligned && onchip_variant() == 0)
                 ? timed("rsum", st, [&] {
                       return launch_rsum(dt, K, x, y, n, w.kglob, w.slots, w.flags, st, &t_launches);
                   })
                 : timed("onchip_accumulate", st, [&] {
                       return launch_onchip_array(dt, K, x, y, n, w.kglob, w.slots, w.flags, st, &t_launches);
                   });
        if (rc) return map_launch(rc);
    }
    if (!(phase & 2)) return REPRO_OK;
    return map_launch(timed("fold", st, [&] {
        return launch_fold(dt, K, 1, w.kglob, w.slots, 0, nullptr, nullptr, nullptr, out, w.flags, st,
                           &t_launches);
    }));
}

int array_blocking(const void *x, const void *y, int64_t n, int32_t fold, int32_t dtype, void *out) {
    t_launches = 0;
    if (n < 0 || !valid_shape(1, fold, dtype) || !out || (n > 0 && !x)) return REPRO_EINVAL;
    const size_t need = repro_dot_workspace_bytes(fold, dtype);
    std::lock_guard<std::mutex> lock(g_cache.mu);
    void *ws = cache_get(need);
    if (!ws) return REPRO_ENOMEM;
    uint32_t *flags = nullptr;
    int rc = enqueue_array(x, y, n, fold, dtype, out, ws, 0, &flags);
    if (rc != REPRO_OK) {
        cudaStreamSynchronize(0);
        return rc;
    }
    return finish_blocking(flags, 0);
}

}  // namespace

extern "C" {

int repro_dot_async(const void *x, const void *y, int64_t n, int32_t fold, int32_t dtype, void *out,
                    void *workspace, size_t ws_bytes, void *stream, int32_t *d_status) {
    t_launches = 0;
    if (n < 0 || !valid_shape(1, fold, dtype) || !out || !workspace || !d_status || (n > 0 && !x))
        return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    if (ws_bytes < repro_dot_workspace_bytes(fold, dtype)) return REPRO_ENOMEM;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *flags = nullptr;
    int rc = enqueue_array(x, y, n, fold, dtype, out, workspace, st, &flags);
    if (rc != REPRO_OK) return rc;
    return map_launch(timed("status", st, [&] { return launch_status(flags, d_status, st, &t_launches); }));
}

int repro_dot_table(int32_t fold, int32_t dtype, int64_t *offsets, int64_t *counts) {
    if (!valid_shape(1, fold, dtype) || !offsets || !counts) return REPRO_EINVAL;
    OnchipWs w = carve_onchip(nullptr, 0, 1, fold, dtype);
    offsets[0] = (int64_t)(uintptr_t)w.flags;
    offsets[1] = (int64_t)(uintptr_t)w.kglob;
    offsets[2] = (int64_t)(uintptr_t)w.slots;
    counts[0] = 1;
    counts[1] = 1;
    counts[2] = (int64_t)slot_count(dtype, fold) * 2;
    return REPRO_OK;
}

int repro_dot_deposit_async(const void *x, const void *y, int64_t n, int32_t fold, int32_t dtype, void *workspace,
                            size_t ws_bytes, void *stream) {
    t_launches = 0;
    if (n < 0 || !valid_shape(1, fold, dtype) || !workspace || (n > 0 && !x)) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    if (ws_bytes < repro_dot_workspace_bytes(fold, dtype)) return REPRO_ENOMEM;
    uint32_t *flags = nullptr;
    return enqueue_array(x, y, n, fold, dtype, nullptr, workspace, (cudaStream_t)stream, &flags, 1);
}

int repro_dot_finish_async(int32_t fold, int32_t dtype, void *out, void *workspace, size_t ws_bytes, void *stream,
                           int32_t *d_status) {
    t_launches = 0;
    if (!valid_shape(1, fold, dtype) || !out || !workspace || !d_status) return REPRO_EINVAL;
    if (((uintptr_t)workspace) % ALIGN) return REPRO_EINVAL;
    if (ws_bytes < repro_dot_workspace_bytes(fold, dtype)) return REPRO_ENOMEM;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *flags = nullptr;
    int rc = enqueue_array(nullptr, nullptr, 0, fold, dtype, out, workspace, st, &flags, 2);
    if (rc != REPRO_OK) return rc;
    return map_launch(timed("status", st, [&] { return launch_status(flags, d_status, st, &t_launches); }));
}

int repro_sum(const void *x, int64_t n, int32_t fold, int32_t dtype, void *out) {
    return array_blocking(x, nullptr, n, fold, dtype, out);
}

int repro_dot(const void *x, const void *y, int64_t n, int32_t fold, int32_t dtype, void *out) {
    if (n > 0 && !y) {
        t_launches = 0;
        return REPRO_EINVAL;
    }
    return array_blocking(x, y, n, fold, dtype, out);
}

// ---- f3: runtime path / depth selection -----------------------------------

int repro_tune_get(int32_t fold, int32_t dtype, int32_t *onchip_max_groups_out, int32_t *onepass_bits_out) {
    if (fold < 1 || fold > 4 || (dtype != REPRO_F32 && dtype != REPRO_F64)) return REPRO_EINVAL;
    if (onchip_max_groups_out) onchip_max_groups_out[0] = g_onchip_cross[dtype == REPRO_F64][fold];
    if (onepass_bits_out) onepass_bits_out[0] = partition_onepass_bits(dtype == REPRO_F64 ? 1 : 0);
    return REPRO_OK;
}

int repro_tune_set(int32_t fold, int32_t dtype, int32_t onchip_max_groups, int32_t onepass_bits) {
    if (fold < 1 || fold > 4 || (dtype != REPRO_F32 && dtype != REPRO_F64)) return REPRO_EINVAL;
    if (onchip_max_groups < 0 || onepass_bits < 0) return REPRO_EINVAL;
    if (onepass_bits > 0 && set_partition_onepass_bits(dtype == REPRO_F64 ? 1 : 0, onepass_bits) != 0)
        return REPRO_EINVAL;
    g_onchip_cross[dtype == REPRO_F64][fold] = onchip_max_groups;
    return REPRO_OK;
}

}  // extern "C"

namespace {

__global__ void k_to_f32(const double *__restrict__ a, float *__restrict__ b, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}

}  // namespace

extern "C" {

int repro_autotune(int64_t n, int32_t fold, int32_t dtype, int32_t *onchip_max_groups_out,
                   int32_t *onepass_bits_out) {
    if (n < (1 << 16) || !valid_shape(1, fold, dtype)) return REPRO_EINVAL;
    n = std::min<int64_t>(n, 1ll << 27);
    const int dt1 = dtype == REPRO_F64 ? 1 : 0;
    const size_t vsz = dtype == REPRO_F64 ? 8 : 4;
    const int cap = onchip_max_groups(fold, dtype);
    const int32_t gmax = std::min<int32_t>(partition_max_groups(fold, dtype), 1 << 20);
    std::lock_guard<std::mutex> lock(g_cache.mu);
    // inputs: config-2 rows (uniform keys, values U[-1,1)) regenerated per G
    int32_t *keys = nullptr;
    double *v64 = nullptr;
    void *vals = nullptr, *out = nullptr, *ws = nullptr;
    size_t wsb = 0;
    for (int32_t G = 2048; G <= gmax; G *= 2)
        wsb = std::max(wsb, std::max(ws_bytes_for(0, n, std::min(G, cap), fold, dtype),
                                     std::max(choose_path(G, fold, dtype) == 1 ? ws_bytes_for(1, n, G, fold, dtype) : 0,
                                              ws_bytes_for(2, n, G, fold, dtype))));
    bool ok = cudaMalloc(&keys, 4 * (size_t)n) == cudaSuccess && cudaMalloc(&v64, 8 * (size_t)n) == cudaSuccess &&
              cudaMalloc(&out, vsz * (size_t)gmax) == cudaSuccess && cudaMalloc(&ws, wsb) == cudaSuccess;
    if (ok && dtype == REPRO_F32) ok = cudaMalloc(&vals, 4 * (size_t)n) == cudaSuccess;
    if (dtype == REPRO_F64) vals = v64;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ok) ok = cudaEventCreate(&e0) == cudaSuccess && cudaEventCreate(&e1) == cudaSuccess;
    const int32_t saved_override = g_path_override;
    const int saved_bits = partition_onepass_bits(dt1);
    auto gen = [&](int32_t G) {
        void *cols[1] = {v64};
        if (launch_synth(2, 0x1802098830ull + 2, 0, n, G, keys, cols, 0) != 0) return false;
        if (dtype == REPRO_F32) k_to_f32<<<4 * device_props().sms, 256>>>(v64, (float *)vals, n);
        return cudaStreamSynchronize(0) == cudaSuccess;
    };
    auto time_path = [&](int32_t G, int path) -> double {  // best of 3, ms; < 0 on error
        g_path_override = path;
        double best = -1;
        for (int r = 0; r < 4; ++r) {
            uint32_t *flags = nullptr;
            cudaEventRecord(e0, 0);
            const int rc = enqueue_groupby(keys, vals, n, G, fold, dtype, out, 0, nullptr, nullptr, nullptr, ws,
                                           wsb, 0, &flags);
            cudaEventRecord(e1, 0);
            if (rc != REPRO_OK || cudaEventSynchronize(e1) != cudaSuccess) return -1;
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && (best < 0 || ms < best)) best = ms;
        }
        return best;
    };
    int32_t cross = 1024;
    int bits = saved_bits;
    const bool tlog = getenv("REPRO_TUNE_LOG") != nullptr;
    if (ok) {
        // (1) on-chip vs partitioned crossover above the register-table size
        bool onchip_wins = true;
        for (int32_t G = 2048; G <= cap && onchip_wins; G *= 2) {
            if (!gen(G)) { ok = false; break; }
            const double a = time_path(G, 0), b = time_path(G, 1);
            if (tlog) fprintf(stderr, "repro_autotune: G=%d on-chip %.3f ms, partitioned %.3f ms\n", G, a, b);
            if (a < 0 || b < 0) { ok = false; break; }
            onchip_wins = a <= b;
            if (onchip_wins) cross = G;
        }
        if (onchip_wins && ok) cross = cap;
        // (2) one vs two scatter passes, partition-id bits 2 .. 10: the
        // threshold T minimising sum_b (b <= T ? one(b) : two(b))
        double one[11] = {}, two[11] = {};
        int bmax = 1;
        for (int b = 2; b <= 10 && ok; ++b) {
            const int64_t G = (int64_t)1024 << b;
            if (G > gmax) break;
            if (!gen((int32_t)G)) { ok = false; break; }
            g_path_override = 2;
            set_partition_onepass_bits(dt1, b);
            one[b] = time_path((int32_t)G, 2);
            set_partition_onepass_bits(dt1, b - 1);
            two[b] = time_path((int32_t)G, 2);
            if (tlog)
                fprintf(stderr, "repro_autotune: G=%lld %d-bit ids: one pass %.3f ms, two passes %.3f ms\n",
                        (long long)G, b, one[b], two[b]);
            if (one[b] < 0 || two[b] < 0) { ok = false; break; }
            bmax = b;
        }
        double best = -1;
        for (int T = 1; T <= bmax && ok; ++T) {
            double c = 0;
            for (int b = 2; b <= bmax; ++b) c += b <= T ? one[b] : two[b];
            if (best < 0 || c < best) {
                best = c;
                bits = T;
            }
        }
        if (bmax < 10 && bits == bmax) bits = saved_bits > bmax ? saved_bits : bits;  // untested widths keep theirs
    }
    g_path_override = saved_override;
    set_partition_onepass_bits(dt1, ok ? std::max(bits, 1) : saved_bits);
    if (ok) g_onchip_cross[dt1][fold] = cross;
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(keys);
    cudaFree(v64);
    if (dtype == REPRO_F32) cudaFree(vals);
    cudaFree(out);
    cudaFree(ws);
    if (!ok) {
        cudaGetLastError();
        return REPRO_ECUDA;
    }
    if (onchip_max_groups_out) onchip_max_groups_out[0] = cross;
    if (onepass_bits_out) onepass_bits_out[0] = partition_onepass_bits(dt1);
    return REPRO_OK;
}

void repro_release_cache(void) {
    {
        std::lock_guard<std::mutex> lock(g_host.mu);
        g_host.release();
    }
    std::lock_guard<std::mutex> lock(g_cache.mu);
    if (g_cache.ptr) cudaFree(g_cache.ptr);
    g_cache.ptr = nullptr;
    g_cache.bytes = 0;
}

// Host-array variant: rows are streamed to the device in chunks on a copy
// stream while the on-chip kernel deposits the previous chunk into the same
// absolute-level slot table (exact whatever the chunking), then one fold.
int repro_groupby_sum_host(const int32_t *keys_host, const void *vals_host, int64_t n, int32_t n_groups,
                           int32_t fold, int32_t dtype, void *out_host) {
    t_launches = 0;
    if (n < 0 || !valid_shape(n_groups, fold, dtype) || !out_host) return REPRO_EINVAL;
    if (n > 0 && (!keys_host || !vals_host)) return REPRO_EINVAL;
    const size_t vsz = dtype == REPRO_F64 ? 8 : 4;
    const int path = choose_path(n_groups, fold, dtype);
    if (path < 0) return REPRO_EINVAL;
    bool pinned_input = false;
    {
        cudaPointerAttributes a{};
        if (n > 0 && cudaPointerGetAttributes(&a, keys_host) == cudaSuccess && a.type == cudaMemoryTypeHost) {
            cudaPointerAttributes b{};
            pinned_input = cudaPointerGetAttributes(&b, vals_host) == cudaSuccess && b.type == cudaMemoryTypeHost;
        }
        cudaGetLastError();
    }
    // on-chip path: chunks of CH rows through NB device buffers; the copy
    // stream waits on the kernel stream only through events (no host sync
    // when the input is pinned), so H2D streams back to back
    const int64_t CH = path == 0 ? ((int64_t)1 << 23) : std::max<int64_t>(n, 1);
    const int nb = path == 0 ? HostCtx::NB : 1;
    const size_t chunk_bytes = align_up((size_t)std::min<int64_t>(CH, std::max<int64_t>(n, 1)) * 4) +
                               (size_t)std::min<int64_t>(CH, std::max<int64_t>(n, 1)) * vsz;
    const size_t need = ws_bytes_for(path, n, n_groups, fold, dtype);
    std::lock_guard<std::mutex> lock(g_host.mu);
    HostCtx &h = g_host;
    int status = h.prepare(chunk_bytes * nb + ALIGN, vsz * (size_t)n_groups, need,
                           pinned_input ? 0 : chunk_bytes);
    if (status != REPRO_OK) return status;
#define CK(x)                                    \
    do {                                         \
        if ((x) != cudaSuccess) {                \
            status = REPRO_ECUDA;                \
            goto done;                           \
        }                                        \
    } while (0)
    if (path == 0) {
        OnchipWs w = carve_onchip(h.ws, n, n_groups, fold, dtype);
        CK(cudaMemsetAsync(h.ws, 0, w.zero_bytes, h.ks));
        int c = 0;
        for (int64_t r0 = 0; r0 < n; r0 += CH, ++c) {
            const int b = c % nb;
            const int64_t rows = std::min<int64_t>(CH, n - r0);
            char *dk = (char *)h.dbuf + (size_t)b * chunk_bytes;
            char *dv = dk + align_up((size_t)rows * 4);
            const char *hk = (const char *)keys_host + (size_t)r0 * 4;
            const char *hv = (const char *)vals_host + (size_t)r0 * vsz;
            if (c >= nb) CK(cudaStreamWaitEvent(h.cs, h.consumed[b], 0));  // device buffer b is free
            if (!pinned_input) {
                // pageable input: stage through one pinned buffer (host waits for its copy)
                CK(cudaStreamSynchronize(h.cs));
                memcpy(h.pin, hk, (size_t)rows * 4);
                memcpy((char *)h.pin + align_up((size_t)rows * 4), hv, (size_t)rows * vsz);
                hk = (const char *)h.pin;
                hv = (const char *)h.pin + align_up((size_t)rows * 4);
            }
            CK(cudaMemcpyAsync(dk, hk, (size_t)rows * 4, cudaMemcpyHostToDevice, h.cs));
            CK(cudaMemcpyAsync(dv, hv, (size_t)rows * vsz, cudaMemcpyHostToDevice, h.cs));
            CK(cudaEventRecord(h.copied[b], h.cs));
            CK(cudaStreamWaitEvent(h.ks, h.copied[b], 0));
            int rc = timed("onchip_accumulate", h.ks, [&] {
                return launch_onchip_any(dtype, fold, (const int32_t *)dk, dv, rows, n_groups, w.kglob, w.slots,
                                         w.flags, h.ks, &t_launches);
            });
            if (rc) { status = map_launch(rc); goto done; }
            CK(cudaEventRecord(h.consumed[b], h.ks));
        }
        int rc = timed("fold", h.ks, [&] {
            return launch_fold(dtype, fold, n_groups, w.kglob, w.slots, 0, nullptr, nullptr, nullptr, h.dout, w.flags,
                               h.ks, &t_launches);
        });
        if (rc) { status = map_launch(rc); goto done; }
        CK(cudaMemcpyAsync(out_host, h.dout, vsz * (size_t)n_groups, cudaMemcpyDeviceToHost, h.ks));
        status = finish_blocking(w.flags, h.ks);
    } else {
        char *dk = (char *)h.dbuf;
        char *dv = dk + align_up((size_t)n * 4);
        CK(cudaMemcpyAsync(dk, keys_host, (size_t)n * 4, cudaMemcpyHostToDevice, h.ks));
        CK(cudaMemcpyAsync(dv, vals_host, (size_t)n * vsz, cudaMemcpyHostToDevice, h.ks));
        uint32_t *flags = nullptr;
        int rc = enqueue_groupby((const int32_t *)dk, dv, n, n_groups, fold, dtype, h.dout, 0, nullptr, nullptr,
                                 nullptr, h.ws, need, h.ks, &flags);
        if (rc != REPRO_OK) { status = rc; goto done; }
        CK(cudaMemcpyAsync(out_host, h.dout, vsz * (size_t)n_groups, cudaMemcpyDeviceToHost, h.ks));
        status = finish_blocking(flags, h.ks);
    }
done:
#undef CK
    cudaStreamSynchronize(h.ks);
    cudaStreamSynchronize(h.cs);
    return status;
}

// ---------------------------------------------------------------------------
// accumulator handles
// ---------------------------------------------------------------------------

int repro_acc_create(repro_acc **acc, int32_t n_groups, int32_t fold, int32_t dtype) {
    t_launches = 0;
    if (!acc || !valid_shape(n_groups, fold, dtype)) return REPRO_EINVAL;
    repro_acc *a = (repro_acc *)calloc(1, sizeof(repro_acc));
    if (!a) return REPRO_ENOMEM;
    a->G = n_groups;
    a->K = fold;
    a->dt = dtype;
    if (cudaMalloc(&a->k, sizeof(int32_t) * (size_t)n_groups) != cudaSuccess ||
        cudaMalloc(&a->C, sizeof(int64_t) * (size_t)n_groups * fold) != cudaSuccess ||
        cudaMalloc(&a->D, sizeof(int64_t) * (size_t)n_groups * fold) != cudaSuccess) {
        cudaGetLastError();
        repro_acc_destroy(a);
        return REPRO_ENOMEM;
    }
    if (launch_reset(fold, n_groups, a->k, a->C, a->D, 0, &t_launches) != 0 || cudaStreamSynchronize(0) != cudaSuccess) {
        repro_acc_destroy(a);
        return REPRO_ECUDA;
    }
    *acc = a;
    return REPRO_OK;
}

void repro_acc_destroy(repro_acc *acc) {
    if (!acc) return;
    if (acc->k) cudaFree(acc->k);
    if (acc->C) cudaFree(acc->C);
    if (acc->D) cudaFree(acc->D);
    free(acc);
}

int32_t repro_acc_n_groups(const repro_acc *acc) { return acc ? acc->G : 0; }
int32_t repro_acc_fold(const repro_acc *acc) { return acc ? acc->K : 0; }
int32_t repro_acc_dtype(const repro_acc *acc) { return acc ? acc->dt : -1; }

int repro_acc_reset(repro_acc *acc) {
    t_launches = 0;
    if (!acc) return REPRO_EINVAL;
    if (launch_reset(acc->K, acc->G, acc->k, acc->C, acc->D, 0, &t_launches) != 0) return REPRO_ECUDA;
    return cudaStreamSynchronize(0) == cudaSuccess ? REPRO_OK : REPRO_ECUDA;
}

int repro_acc_deposit(repro_acc *acc, const int32_t *keys, const void *vals, int64_t n) {
    t_launches = 0;
    if (!acc || n < 0 || (n > 0 && (!keys || !vals))) return REPRO_EINVAL;
    if (n == 0) return REPRO_OK;
    const size_t need = repro_groupby_workspace_bytes(n, acc->G, acc->K, acc->dt);
    if (need == 0) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    void *ws = cache_get(need);
    if (!ws) return REPRO_ENOMEM;
    uint32_t *flags = nullptr;
    int rc = enqueue_groupby(keys, vals, n, acc->G, acc->K, acc->dt, nullptr, 1, acc->k, acc->C, acc->D, ws, need, 0,
                             &flags);
    if (rc != REPRO_OK) {
        cudaStreamSynchronize(0);
        return rc;
    }
    return finish_blocking(flags, 0);
}

static int run_small(int launch_rc, uint32_t *flags) {
    if (launch_rc) {
        cudaStreamSynchronize(0);
        return map_launch(launch_rc);
    }
    return finish_blocking(flags, 0);
}

static uint32_t *small_flags() {
    void *ws = cache_get(ALIGN);
    if (!ws) return nullptr;
    if (cudaMemsetAsync(ws, 0, sizeof(uint32_t), 0) != cudaSuccess) return nullptr;
    return (uint32_t *)ws;
}

int repro_acc_merge(repro_acc *dst, const repro_acc *src) {
    t_launches = 0;
    if (!dst || !src || dst->G != src->G || dst->K != src->K || dst->dt != src->dt) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    uint32_t *f = small_flags();
    if (!f) return REPRO_ENOMEM;
    return run_small(launch_merge_state(dst->dt, dst->K, dst->G, dst->k, dst->C, dst->D, src->k, src->C, src->D, f, 0,
                                        &t_launches),
                     f);
}

int repro_acc_finalize(const repro_acc *acc, void *out) {
    t_launches = 0;
    if (!acc || !out) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    uint32_t *f = small_flags();
    if (!f) return REPRO_ENOMEM;
    return run_small(launch_finalize(acc->dt, acc->K, acc->G, acc->k, acc->C, acc->D, out, f, 0, &t_launches), f);
}

int repro_acc_export(const repro_acc *acc, void *state) {
    t_launches = 0;
    if (!acc || !state) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    uint32_t *f = small_flags();
    if (!f) return REPRO_ENOMEM;
    return run_small(launch_export(acc->dt, acc->K, acc->G, acc->k, acc->C, acc->D, state, f, 0, &t_launches), f);
}

int repro_acc_import(repro_acc *acc, const void *state) {
    t_launches = 0;
    if (!acc || !state) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    uint32_t *f = small_flags();
    if (!f) return REPRO_ENOMEM;
    return run_small(launch_import(acc->dt, acc->K, acc->G, state, acc->k, acc->C, acc->D, f, 0, &t_launches), f);
}

int repro_acc_top_levels(const repro_acc *acc, int32_t *k_out) {
    t_launches = 0;
    if (!acc || !k_out) return REPRO_EINVAL;
    if (cudaMemcpyAsync(k_out, acc->k, sizeof(int32_t) * (size_t)acc->G, cudaMemcpyDeviceToDevice, 0) != cudaSuccess)
        return REPRO_ECUDA;
    return cudaStreamSynchronize(0) == cudaSuccess ? REPRO_OK : REPRO_ECUDA;
}

int repro_acc_window_export(const repro_acc *acc, const int32_t *k_global, int64_t *limbs_out) {
    t_launches = 0;
    if (!acc || !k_global || !limbs_out) return REPRO_EINVAL;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    uint32_t *f = small_flags();
    if (!f) return REPRO_ENOMEM;
    return run_small(launch_window_export(acc->dt, acc->K, acc->G, acc->k, acc->C, acc->D, k_global, limbs_out, f, 0,
                                          &t_launches),
                     f);
}

int repro_acc_window_import_range(repro_acc *acc, int32_t g0, int32_t count, const int32_t *k_global,
                                  const int64_t *limbs) {
    t_launches = 0;
    if (!acc || !k_global || !limbs || g0 < 0 || count < 0 || (int64_t)g0 + count > acc->G) return REPRO_EINVAL;
    if (count == 0) return REPRO_OK;
    int rc = launch_window_import(acc->dt, acc->K, count, k_global, limbs, acc->k + g0, acc->C + (size_t)g0 * acc->K,
                                  acc->D + (size_t)g0 * acc->K, nullptr, 0, &t_launches);
    if (rc) return map_launch(rc);
    return cudaStreamSynchronize(0) == cudaSuccess ? REPRO_OK : REPRO_ECUDA;
}

int repro_acc_window_import(repro_acc *acc, const int32_t *k_global, const int64_t *limbs) {
    if (!acc) return REPRO_EINVAL;
    return repro_acc_window_import_range(acc, 0, acc->G, k_global, limbs);
}

int repro_baseline_atomic_sum(const int32_t *keys, const void *vals, int64_t n, int32_t n_groups, int32_t dtype,
                              int32_t variant, int32_t accumulate_f64, void *out, void *stream) {
    t_launches = 0;
    if (n < 0 || n_groups < 1 || (dtype != 0 && dtype != 1) || !out || (n > 0 && (!keys || !vals)))
        return REPRO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    static const char *names[5] = {"baseline_atomic_global", "baseline_atomic_smem", "baseline_atomic_regs",
                                   "baseline_atomic_match", "baseline_atomic_heavy"};
    if (variant < 0 || variant > 4) return REPRO_EINVAL;
    return map_launch(timed(names[variant], st, [&] {
        return launch_baseline(dtype, variant, accumulate_f64, keys, vals, n, n_groups, out, st, &t_launches);
    }));
}

}  // extern "C"
