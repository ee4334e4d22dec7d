// internal.h -- host-side declarations shared by the .cu files of the library
// (not part of the C-ABI; see include/repro_groupby.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace repro {

struct DeviceProps {
    int device;
    int sms;
    int smem_optin;  // max dynamic shared memory per block (opt-in)
};
const DeviceProps &device_props();

// Number of absolute lattice slots of a group's slot table: levels
// -(K-1) .. KMAX, slot = level + K - 1.
inline int slot_count(int DT, int K) { return (DT == 1 ? 25 : 7) + K; }

// measured add rate of the FP pipe of `DT` on this GPU (k_peak.cu)
int measure_fp_add_rate(int DT, double *adds_per_s, cudaStream_t st);

// ---- launchers (return 0 on success, -1 unsupported shape, -2 CUDA error) --
int onchip_max_groups(int K, int DT);
void set_onchip_variant(int v);
int onchip_variant();  // 0 auto, 1 atomic (TMA ring), 2 table (k_table.cu), 3 atomic + register loads
int atomic_max_groups(int K, int DT);
int table_max_groups(int K, int DT);
int launch_table_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G,
                     int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                     int *launches);
int launch_atomic_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G,
                      int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                      int *launches);
int launch_onchip_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G,
                      int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                      int *launches);

// multi-column on-chip GroupBy (k_onchip.cu): virtual columns per group for a
// (proj, ncols) shape (-1: no fused kernel), and the launcher over G real
// groups (virtual groups j * G + g; -1 if this shape cannot run fused)
int multi_virtual_columns(int proj, int ncols);
int launch_rsum(int DT, int K, const void *x, const void *y, int64_t n, int32_t *kglob, unsigned long long *slots,
                uint32_t *status, cudaStream_t st, int *launches);
int launch_onchip_array(int DT, int K, const void *x, const void *y, int64_t n, int32_t *kglob,
                        unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches);
bool lean_single_applies(const int32_t *keys, const void *vals, int32_t G);
int launch_lean_single(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t *kglob,
                       unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches);
bool lean_multi_applies(int DT, int proj, int ncols, const int32_t *keys, const void *const *cols, int32_t G);
int launch_lean_multi(int DT, int K, int proj, int ncols, const int32_t *keys, const void *const *cols, int64_t n,
                      int32_t G, int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                      int *launches);
int launch_onchip_multi(int DT, int K, int proj, int ncols, const int32_t *keys, const void *const *cols, int64_t n,
                        int32_t G, int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                        int *launches);

int launch_multi_scatter(int DT, int K, const void *vout, int32_t G, int nsum, void *const *outs,
                         const unsigned long long *slots, int64_t *counts, cudaStream_t st, int *launches);
int launch_q1_project(const double *price, const double *disc, const double *tax, int64_t n, double *dp,
                      double *charge, cudaStream_t st, int *launches);
int launch_count_rows(const int32_t *keys, int64_t n, int32_t G, int64_t *counts, cudaStream_t st, int *launches);
int launch_flags_or(uint32_t *acc, const uint32_t *f, cudaStream_t st, int *launches);
int launch_square(int DT, const void *x, int64_t n, void *sq, cudaStream_t st, int *launches);
int launch_moments(int DT, const void *s, const void *q, const int64_t *cnt, int32_t G, void *avg, void *var, void *sd,
                   cudaStream_t st, int *launches);

// arbitrary int64 / int32 keys -> dense ids (k_sparse.cu)
uint64_t sparse_table_slots(int64_t max_groups);
size_t sparse_scratch_bytes(int64_t n, int64_t max_groups);
template <typename KeyT>
int sparse_map_keys(const KeyT *keys, int64_t n, int64_t max_groups, void *scratch, int64_t *sorted_out,
                    int32_t **ids_out, int64_t *d_out, uint32_t *status, cudaStream_t st, int *launches);

// device copy of synth.py's seeded generator (bench/test support, k_synth.cu)
int launch_synth(int config, uint64_t seed, int64_t r0, int64_t n, int32_t G, int32_t *keys, void *const *cols,
                 cudaStream_t st);

// slots (+ global tops) -> canonical state; optionally merged with the
// existing state (acc_*), optionally finalised into out.  `merge` != 0 reads
// acc_k/acc_C/acc_D as the previous state.
int launch_fold(int DT, int K, int32_t G, const int32_t *kglob, const unsigned long long *slots,
                int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out,
                uint32_t *status, cudaStream_t st, int *launches);

// multi-GPU exchange of the slot table: K slot words under the global tops,
// and the read-out of a group range from summed limbs
int launch_slot_limbs(int DT, int K, int32_t G, const int32_t *kg, const unsigned long long *slots, int64_t *limbs,
                      cudaStream_t st, int *launches);
int launch_limbs_finalize(int DT, int K, int32_t count, const int32_t *kg, const int64_t *limbs, void *out,
                          uint32_t *status, cudaStream_t st, int *launches);

// canonical state -> Eq. 1 read-out
int launch_finalize(int DT, int K, int32_t G, const int32_t *k, const int64_t *C, const int64_t *D,
                    void *out, uint32_t *status, cudaStream_t st, int *launches);
int launch_export(int DT, int K, int32_t G, const int32_t *k, const int64_t *C, const int64_t *D,
                  void *state, uint32_t *status, cudaStream_t st, int *launches);
int launch_import(int DT, int K, int32_t G, const void *state, int32_t *k, int64_t *C, int64_t *D,
                  uint32_t *status, cudaStream_t st, int *launches);
int launch_merge_state(int DT, int K, int32_t G, int32_t *dk, int64_t *dC, int64_t *dD,
                       const int32_t *sk, const int64_t *sC, const int64_t *sD, uint32_t *status,
                       cudaStream_t st, int *launches);
int launch_reset(int K, int32_t G, int32_t *k, int64_t *C, int64_t *D, cudaStream_t st, int *launches);
int launch_window_export(int DT, int K, int32_t G, const int32_t *k, const int64_t *C,
                         const int64_t *D, const int32_t *kg, int64_t *limbs, uint32_t *status,
                         cudaStream_t st, int *launches);
int launch_window_import(int DT, int K, int32_t count, const int32_t *kg, const int64_t *limbs,
                         int32_t *k, int64_t *C, int64_t *D, uint32_t *status, cudaStream_t st,
                         int *launches);
int launch_status(const uint32_t *flags, int32_t *d_status, cudaStream_t st, int *launches);

// ---- per-kernel event timing (repro_timing_enable) ------------------------
// trace_begin returns a token (or -1 when timing is off); trace_end records
// the kernel named `name` between the two events on `st`.
int trace_begin(cudaStream_t st);
void trace_end(int token, const char *name, cudaStream_t st);

// ---- partitioned (high-cardinality) path --------------------------------
int partition_max_groups(int K, int DT);
int partition_onepass_bits(int DT);             // f3: partitioning depth setting
int set_partition_onepass_bits(int DT, int bits);
size_t partition_workspace_bytes(int64_t n, int32_t G, int K, int DT);
int launch_partitioned(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G,
                       void *ws, size_t ws_bytes, int merge, int32_t *acc_k, int64_t *acc_C,
                       int64_t *acc_D, void *out, uint32_t *status, cudaStream_t st, int *launches);

// ---- partitioned path: two-pass sweep (k_sweep.cu) ----------------------
int sweep_max_groups(int K, int DT);
size_t sweep_workspace_bytes(int64_t n, int32_t G, int K, int DT);
int launch_sweep(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws,
                 size_t ws_bytes, int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out,
                 uint32_t *status, cudaStream_t st, int *launches);

// ---- routed one-pass path (k_route.cu): rows move to their group's SM
// through L2 rings; -1 when the shape does not apply (the sweep runs)
void set_route_mode(int m);  // 0 off, 1 auto
int route_mode();
size_t route_workspace_bytes(int32_t G, int K, int DT);
int launch_route(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G, void *ws,
                 size_t ws_bytes, int merge, int32_t *acc_k, int64_t *acc_C, int64_t *acc_D, void *out,
                 uint32_t *status, cudaStream_t st, int *launches);

// ---- NVLS (multimem) all-reduce of a slot table (k_nvls.cu) --------------
int launch_nvls_reduce(uint32_t *mc_flags, int32_t *mc_kglob, int64_t nk, unsigned long long *mc_slots, int64_t ns,
                       int rank, int world, cudaStream_t st, int *launches);

// ---- non-reproducible baseline --------------------------------------------
int launch_baseline(int DT, int variant, int acc64, const int32_t *keys, const void *vals,
                    int64_t n, int32_t G, void *out, cudaStream_t st, int *launches);

}  // namespace repro
