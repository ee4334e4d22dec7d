/*
 * repro_groupby.h -- C-ABI of the B200-native reproducible GroupBy-SUM
 * (arxiv 1802.09883, "Reproducible Floating-Point Aggregation in RDBMSs").
 *
 * The operation (Section 2.1): turn a sequence of
 * <key, value> pairs into <key, aggregate> pairs, where the aggregate of a
 * group is the sum of its values, with "exactly the same bit pattern for any
 * execution".  Each group's sum is the paper's repro<ScalarT, L> accumulator
 * with L = `fold` levels: Algorithm 1
 * deposits, operator+=(repro) merges,
 * Eq. 1 reads out.  Readings where the paper is silent
 * (ties away from zero, threshold 2^(W-1) ulp, f = 0, W = 40 / 18) are listed
 * in DESIGN.md; the result bits equal those of the CPU oracle in oracle/.
 *
 * Conventions shared by every entry point
 *   - Array arguments are CUDA DEVICE pointers owned by the caller, unless the
 *     name ends in _host.  Keys are int32, dense in [0, n_groups) (identity
 *     hashing).  Values are binary32 (dtype REPRO_F32) or
 *     binary64 (REPRO_F64); `out` has n_groups elements of the same type.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Blocking calls return after the stream has been synchronised and report
 *     device-detected errors.  _async calls only enqueue work; their device
 *     status word (int32, device memory, caller owned) receives the status.
 *   - Argument errors (REPRO_EINVAL) are reported before anything is
 *     launched: n < 0, n_groups < 1, fold not in [1, 4],
 *     unknown dtype, NULL pointer with n > 0, mismatched accumulators.
 *   - Device-detected errors have a fixed precedence that does not depend on
 *     row order: REPRO_EKEY (key outside [0, n_groups)) > REPRO_EDOM (NaN or
 *     Inf value) > REPRO_ERANGE (|value| >= 2^987 for binary64 / 2^120 for
 *     binary32, where the top extractor would overflow; or a binary32 carry
 *     count |C| >= 2^24 at read-out).  Output contents are unspecified on
 *     error.
 *   - Empty groups and exactly cancelling groups read out as +0.0.
 *   - Guarantee: `out` bits depend only on the multiset of (key, value)
 *     pairs, fold and dtype -- not on row order, chunking into deposits,
 *     merge order, launch configuration or GPU count.
 */
#ifndef REPRO_GROUPBY_H
#define REPRO_GROUPBY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype */
#define REPRO_F32 0 /* binary32: m = 23, W = 18 */
#define REPRO_F64 1 /* binary64: m = 52, W = 40                     */

/* status codes */
#define REPRO_OK 0
#define REPRO_EINVAL (-1)
#define REPRO_EKEY (-2)
#define REPRO_EDOM (-3)
#define REPRO_ERANGE (-4)
#define REPRO_ECUDA (-5)
#define REPRO_ENOMEM (-6)

/* Human-readable name of a status code (static string). */
const char *repro_strerror(int status);

/* Library build/version string (static). */
const char *repro_version(void);

/* ------------------------------------------------------------------------
 * One-shot GroupBy-SUM
 * ---------------------------------------------------------------------- */

/* out[g] = reproducible sum of vals[i] over rows with keys[i] == g,
 * for g in [0, n_groups).  keys: int32[n]; vals: dtype[n]; out: dtype[n_groups].
 * Blocking; scratch memory comes from a library-internal cache (grown on
 * demand, freed by repro_release_cache). */
int repro_groupby_sum(const int32_t *keys, const void *vals, int64_t n,
                      int32_t n_groups, int32_t fold, int32_t dtype, void *out);

/* Bytes of device workspace repro_groupby_sum_async needs for this shape. */
size_t repro_groupby_workspace_bytes(int64_t n, int32_t n_groups, int32_t fold,
                                     int32_t dtype);

/* Enqueue the GroupBy-SUM on `stream` using the caller's workspace
 * (>= repro_groupby_workspace_bytes, 256-byte aligned).  d_status: int32 in
 * device memory, overwritten with the REPRO_* status when the work completes.
 * Returns REPRO_EINVAL / REPRO_ENOMEM (workspace too small) / REPRO_ECUDA at
 * enqueue time, else REPRO_OK. */
int repro_groupby_sum_async(const int32_t *keys, const void *vals, int64_t n,
                            int32_t n_groups, int32_t fold, int32_t dtype,
                            void *out, void *workspace, size_t ws_bytes,
                            void *stream, int32_t *d_status);

/* Same result from HOST arrays (pageable or pinned): the library copies the
 * rows to the device in pipelined chunks overlapped with the deposit
 * kernels, and copies out[n_groups] back.  Blocking. */
int repro_groupby_sum_host(const int32_t *keys_host, const void *vals_host,
                           int64_t n, int32_t n_groups, int32_t fold,
                           int32_t dtype, void *out_host);

/* Free the internal workspace cache of the blocking entry points. */
void repro_release_cache(void);

/* Split form of repro_groupby_sum for several GPUs (SURVEY.md 8(e) steps
 * 1-5), stream-ordered end to end (no host synchronisation); only for group
 * counts the on-chip table or the two-pass sweep covers (n_groups <=
 * repro_sweep_max_groups), else REPRO_EINVAL.  Workspace: as for
 * repro_groupby_sum_async.
 *  - repro_groupby_table: byte offsets (from the workspace start) and element
 *    counts of the status word (uint32[1]), the global tops kglob (int32[G])
 *    and the ABSOLUTE-LEVEL slot table (uint64[G][fold + 25 or + 7][2], used
 *    as int64) that a deposit leaves in the workspace.
 *  - repro_groupby_deposit_async: zero the table and deposit this rank's rows
 *    (status bits EKEY/EDOM/ERANGE of the rows in the status word).
 *  Exchange A (any n_groups): all-reduce the status word with bitwise OR
 *  (e.g. MAX per bit), kglob with MAX and the slot table with SUM, then
 *  repro_groupby_finish_async on every rank: Eq. 1 of every group into
 *  out[n_groups], status into *d_status.
 *  Exchange B (reduce-scatter by group range): all-reduce the status bits and
 *  kglob (MAX); repro_groupby_window_limbs_async writes, per group, the fold
 *  slot words under the global top k_global[g] (the paper's demotion,
 *  PAPER.md:660-665, is a choice of slots) to limbs int64[G][fold][2]; the
 *  caller reduce-scatters the limbs with SUM by contiguous group range and
 *  each rank calls repro_groupby_finish_limbs_async for its range [g0, g0 +
 *  count) (k_range = k_global + g0, limbs_range and out_range indexed from
 *  g0); the caller all-gathers the outputs.  Integer SUM / MAX only, so the
 *  bits equal repro_groupby_sum's for any rank count and reduction order. */
int repro_groupby_table(int64_t n, int32_t n_groups, int32_t fold, int32_t dtype,
                        int64_t *offsets, int64_t *counts);

/* Exchange A through the switch (NVLS): the workspace
 * lives in symmetric memory that every rank also maps at one MULTICAST
 * address (mc_workspace: the multicast address of the 256-byte aligned
 * workspace start).  offsets / counts: the 3 regions of repro_groupby_table
 * (or repro_groupby_multi_table / repro_dot_table): status word, kglob,
 * slots.  Rank `rank` of `world` reduces its 1/world slice of each region
 * with multimem.ld_reduce (OR / MAX / integer ADD) and multimem-stores the
 * result to every rank.  The caller brackets the call with barriers across
 * the ranks (all deposits done before; all stores visible after), then
 * finishes as for exchange A.  Stream-ordered. */
int repro_nvls_table_allreduce_async(void *mc_workspace, const int64_t *offsets,
                                     const int64_t *counts, int32_t rank,
                                     int32_t world, void *stream);
int repro_groupby_deposit_async(const int32_t *keys, const void *vals, int64_t n,
                                int32_t n_groups, int32_t fold, int32_t dtype,
                                void *workspace, size_t ws_bytes, void *stream);
int repro_groupby_finish_async(int64_t n, int32_t n_groups, int32_t fold,
                               int32_t dtype, void *out, void *workspace,
                               size_t ws_bytes, void *stream, int32_t *d_status);
int repro_groupby_window_limbs_async(int64_t n, int32_t n_groups, int32_t fold,
                                     int32_t dtype, const int32_t *k_global,
                                     int64_t *limbs, void *workspace,
                                     size_t ws_bytes, void *stream);
int repro_groupby_finish_limbs_async(int64_t n, int32_t n_groups, int32_t fold,
                                     int32_t dtype, int32_t g0, int32_t count,
                                     const int32_t *k_range,
                                     const int64_t *limbs_range, void *out_range,
                                     void *workspace, size_t ws_bytes,
                                     void *stream, int32_t *d_status);

/* Split form of the fused multi-column call for several GPUs (SURVEY.md
 * 8(e)); only for shapes the fused pass covers (n_groups * (outputs + 1) <=
 * 1024), else REPRO_EINVAL.  Each rank deposits its rows into the absolute-
 * level slot table inside its workspace (same workspace size as
 * repro_groupby_sum_multi_async), the caller all-reduces that table across
 * the ranks -- the status word with bitwise OR, kglob (int32) with MAX, slots
 * (uint64, used as int64) with SUM: integer operations, so the result does not
 * depend on the reduction order -- and every rank finishes: Eq. 1 read-out of
 * the summed table, scatter to outs / counts, device status word.
 * repro_groupby_multi_table gives the byte offsets inside the workspace and
 * the element counts of [flags (uint32), kglob (int32), slots (uint64)]. */
int repro_groupby_multi_table(int64_t n, int32_t n_groups, int32_t ncols,
                              int32_t proj, int32_t fold, int32_t dtype,
                              int64_t *offsets, int64_t *counts);
int repro_groupby_multi_deposit_async(const int32_t *keys,
                                      const void *const *cols, int32_t ncols,
                                      int32_t proj, int64_t n, int32_t n_groups,
                                      int32_t fold, int32_t dtype,
                                      void *workspace, size_t ws_bytes,
                                      void *stream);
int repro_groupby_multi_finish_async(int64_t n, int32_t n_groups, int32_t ncols,
                                     int32_t proj, int32_t fold, int32_t dtype,
                                     void *const *outs, int64_t *counts,
                                     void *workspace, size_t ws_bytes,
                                     void *stream, int32_t *d_status);

/* Bench / test support, not part of the method: the seeded synthetic input
 * generator of paper_1802_09883_b200/synth.py run on the device (rows r0 ..
 * r0+n of BASELINE config 0/1/2 -- one binary64 column -- or 4 -- columns
 * qty, price, disc, tax), bit-identical to the numpy generator.  keys int32[n],
 * cols: HOST array of DEVICE pointers.  Stream-ordered; EINVAL for other
 * configs. */
int repro_synth_generate(int32_t config, uint64_t seed, int64_t r0, int64_t n,
                         int32_t n_groups, int32_t *keys, void *const *cols,
                         void *stream);

/* ------------------------------------------------------------------------
 * Several aggregates of one key column in one pass
 * ---------------------------------------------------------------------- */

/* Multi-column GroupBy: SUMs of several value columns plus COUNT, grouped by
 * one key column (the paper reduces every SQL float aggregate to SUM,
 * PAPER.md:163-174; the aggregation-heavy query shape of its TPC-H Q1
 * experiment, stood in for by BASELINE config 4).
 *   cols:  HOST array of ncols DEVICE pointers, each dtype[n].
 *   proj:  0 -- outs[c][g] = reproducible sum of cols[c] over group g
 *             (ncols in [1, 8], binary32 or binary64);
 *          2 -- second moments (ncols == 1, column x): outs[0] = SUM(x),
 *             outs[1] = SUM(x * x), each square rounded once;
 *          1 -- the config-4 projection (binary64 only, ncols == 4, columns
 *             qty, price, disc, tax): outs[0] = SUM(qty), outs[1] =
 *             SUM(price), outs[2] = SUM(price * (1 - disc)), outs[3] =
 *             SUM(price * (1 - disc) * (1 + tax)), every product and
 *             difference rounded separately to binary64 (no FMA; DESIGN.md
 *             reading A-15).
 *   outs:  HOST array of (proj 1: 4, proj 2: 2, else ncols) DEVICE
 *          pointers, dtype[n_groups].
 *   counts: DEVICE int64[n_groups] (exact row counts per group) or NULL.
 * Each SUM has the bits repro_groupby_sum would give on that column; rows
 * with a bad key raise REPRO_EKEY for the whole call.  One fused pass when
 * n_groups * (outputs + 1) <= 1024 (the aggregates become virtual groups of
 * one on-chip table), otherwise one pass per output column.  Blocking. */
int repro_groupby_sum_multi(const int32_t *keys, const void *const *cols,
                            int32_t ncols, int32_t proj, int64_t n,
                            int32_t n_groups, int32_t fold, int32_t dtype,
                            void *const *outs, int64_t *counts);

/* GroupBy-SUM over ARBITRARY int64 keys (the paper's
 * operators hash keys): the keys are mapped to dense ids
 * through a GPU hash table (open addressing, 2^b >= 2 max_groups slots), the
 * distinct keys are sorted ascending, and the dense reproducible GroupBy runs
 * on the ids.  Outputs: out_keys[0..d) = the distinct keys ascending,
 * out_vals[0..d) = their reproducible sums (dtype), *n_groups_out = d.  Both
 * depend only on the multiset of (key, value) pairs.  keys: DEVICE int64[n]
 * (INT64_MIN is reserved: REPRO_EKEY); out_keys / out_vals: DEVICE arrays of
 * max_groups elements.  More than max_groups distinct keys: REPRO_ENOMEM with
 * *n_groups_out = the distinct count (retry with a larger capacity).  max_groups
 * is limited by the dense path (2^26).  Blocking. */
int repro_groupby_sum_sparse(const int64_t *keys, const void *vals, int64_t n,
                             int64_t max_groups, int32_t fold, int32_t dtype,
                             int64_t *out_keys, void *out_vals,
                             int64_t *n_groups_out);

/* The same over ARBITRARY int32 keys (every int32 value is a valid key;
 * out_keys are the distinct keys ascending, sign-extended to int64).  keys:
 * DEVICE int32[n].  Same outputs, errors and blocking as above. */
int repro_groupby_sum_sparse_i32(const int32_t *keys, const void *vals, int64_t n,
                                 int64_t max_groups, int32_t fold, int32_t dtype,
                                 int64_t *out_keys, void *out_vals,
                                 int64_t *n_groups_out);

/* AVG / sample VARIANCE / STDDEV per group from reproducible SUMs (SURVEY.md
 * 8(f) f2; the paper reduces every float aggregate to SUM):
 * one fused pass computes SUM(x), SUM(x*x) and COUNT (proj 2 above), then,
 * per group with c = COUNT, s = SUM(x), q = SUM(x*x), each operation rounded
 * once in this order: avg = s / c; var = max(0, (q - (s * s) / c) / (c - 1))
 * (0 when c <= 1); stddev = sqrt(var); an empty group gives avg = 0.  Every
 * output is therefore exactly as reproducible as the SUMs.  sum, avg, var,
 * stddev: DEVICE dtype[n_groups] (avg / var / stddev may be NULL); counts:
 * DEVICE int64[n_groups] (required).  Blocking. */
int repro_groupby_moments(const int32_t *keys, const void *vals, int64_t n,
                          int32_t n_groups, int32_t fold, int32_t dtype,
                          void *sum, void *avg, void *var, void *stddev,
                          int64_t *counts);

/* Workspace bytes of repro_groupby_sum_multi_async (0 on invalid shape). */
size_t repro_groupby_multi_workspace_bytes(int64_t n, int32_t n_groups,
                                           int32_t ncols, int32_t proj,
                                           int32_t fold, int32_t dtype);

/* Stream-ordered form with the caller's workspace and device status word
 * (conventions of repro_groupby_sum_async). */
int repro_groupby_sum_multi_async(const int32_t *keys, const void *const *cols,
                                  int32_t ncols, int32_t proj, int64_t n,
                                  int32_t n_groups, int32_t fold,
                                  int32_t dtype, void *const *outs,
                                  int64_t *counts, void *workspace,
                                  size_t ws_bytes, void *stream,
                                  int32_t *d_status);

/* ------------------------------------------------------------------------
 * Keyless single-array reproducible SUM and dot product (SURVEY.md 8(f) f4:
 * the RSum algorithm's original setting, one group -- PAPER.md:755-757; the
 * K-fold accumulator of Alg. 1, finalised by Eq. 1,
 * PAPER.md:695-702).  x, y: DEVICE dtype[n], any alignment; the dot product
 * deposits x[i] (x) y[i] (one rounding per product, reading A-19 of
 * DESIGN.md).  out: DEVICE dtype[1].  The result is the same bits as
 * repro_groupby_sum with every key 0 over x (or over the products), for any
 * order, launch geometry or GPU count.  Status codes as repro_groupby_sum
 * (NaN/Inf -> REPRO_EDOM; out then holds the IEEE sum of the specials).
 * n == 0 writes +0.
 * ---------------------------------------------------------------------- */
int repro_sum(const void *x, int64_t n, int32_t fold, int32_t dtype, void *out);
int repro_dot(const void *x, const void *y, int64_t n, int32_t fold,
              int32_t dtype, void *out);

/* Workspace bytes of repro_dot_async (0 on invalid fold / dtype). */
size_t repro_dot_workspace_bytes(int32_t fold, int32_t dtype);

/* Stream-ordered SUM (y == NULL) or dot product with the caller's workspace
 * (>= repro_dot_workspace_bytes, 256-byte aligned) and device status word
 * (conventions of repro_groupby_sum_async). */
int repro_dot_async(const void *x, const void *y, int64_t n, int32_t fold,
                    int32_t dtype, void *out, void *workspace,
                    size_t ws_bytes, void *stream, int32_t *d_status);

/* Multi-GPU split form of repro_dot_async (conventions of the
 * repro_groupby_multi_* split form): repro_dot_table gives the byte offsets
 * (from the 256-aligned workspace start) and element counts of the status
 * word (int32[1]), the window top (int32[1]) and the absolute-level slot
 * table (int64[2 * (KMAX + fold)]); after repro_dot_deposit_async on every
 * rank, all-reduce them (status bits OR, top MAX, slots SUM -- integer
 * operations, any order) and call repro_dot_finish_async. */
int repro_dot_table(int32_t fold, int32_t dtype, int64_t *offsets,
                    int64_t *counts);
int repro_dot_deposit_async(const void *x, const void *y, int64_t n,
                            int32_t fold, int32_t dtype, void *workspace,
                            size_t ws_bytes, void *stream);
int repro_dot_finish_async(int32_t fold, int32_t dtype, void *out,
                           void *workspace, size_t ws_bytes, void *stream,
                           int32_t *d_status);

/* ------------------------------------------------------------------------
 * Runtime path / depth selection (the paper picks the
 * partitioning depth offline and names adaptive selection, PAPER.md:
 * 1155-1176).  Every path and depth returns the same bits, so these settings
 * change speed only.  They are process-wide (not thread-safe against
 * concurrent calls) and take effect at the next call; workspace sizes
 * (repro_*_workspace_bytes) must be re-queried after a change, since the
 * on-chip and partitioned paths need different workspaces (a workspace too
 * small for the chosen path gives REPRO_ENOMEM, never a wrong result).
 * ---------------------------------------------------------------------- */

/* Current settings for (fold, dtype): the group count up to which the
 * on-chip path is used (0 = up to its capacity, repro_onchip_max_groups)
 * and the widest partition id (bits) scattered in ONE pass (wider ids take
 * two passes).  Either output pointer may be NULL.  Host-only call. */
int repro_tune_get(int32_t fold, int32_t dtype,
                   int32_t *onchip_max_groups_out, int32_t *onepass_bits_out);

/* Set them: onchip_max_groups >= 0 (0 = capacity; values above the capacity
 * act as the capacity), onepass_bits in 1..10 (0 = leave unchanged).
 * REPRO_EINVAL otherwise.  Host-only call. */
int repro_tune_set(int32_t fold, int32_t dtype, int32_t onchip_max_groups,
                   int32_t onepass_bits);

/* Measure the crossovers on this GPU and set them: (1) the largest group
 * count (powers of two from 2048 up to the on-chip capacity) at which the
 * on-chip path is not slower than the partitioned one, (2) the largest
 * partition-id width (2..10 bits) at which one scatter pass is not slower
 * than two.  Inputs are n (clamped to [2^16, 2^27]) device-generated rows
 * shaped like BASELINE config 2 (uniform keys, values in [-1, 1)).
 * Blocking; allocates and frees its own device memory.  Outputs may be
 * NULL.  REPRO_EINVAL for n < 2^16 or a bad fold / dtype. */
int repro_autotune(int64_t n, int32_t fold, int32_t dtype,
                   int32_t *onchip_max_groups_out, int32_t *onepass_bits_out);

/* ------------------------------------------------------------------------
 * Accumulator handles: n_groups device-resident repro<ScalarT, fold> states
 * (the paper's intermediate aggregates).  A handle is not
 * thread-safe; distinct handles are independent.  All calls are blocking.
 * ---------------------------------------------------------------------- */
typedef struct repro_acc repro_acc;

/* New handle with every group at the initial state (O1). */
int repro_acc_create(repro_acc **acc, int32_t n_groups, int32_t fold,
                     int32_t dtype);

/* Deposit n rows (device arrays) into the handle (Alg. 1 per row). */
int repro_acc_deposit(repro_acc *acc, const int32_t *keys, const void *vals,
                      int64_t n);

/* dst += src (operator+=(repro)); same shape required;
 * dst == src doubles the state. */
int repro_acc_merge(repro_acc *dst, const repro_acc *src);

/* out[g] = Eq. 1 read-out of every group (device array); non-mutating. */
int repro_acc_finalize(const repro_acc *acc, void *out);

/* Serialised state: per group S[0..fold) then C[0..fold) in
 * the native width (double for F64, float for F32), little-endian; device
 * array of n_groups * 2 * fold elements.  Non-mutating. */
int repro_acc_export(const repro_acc *acc, void *state);

/* Replace the handle's state by a serialised one (REPRO_EINVAL if any group
 * is not a canonical state: S off the W-lattice, S outside [1.5, 1.75) ufp,
 * C not an integer). */
int repro_acc_import(repro_acc *acc, const void *state);

/* Reset every group to the initial state. */
int repro_acc_reset(repro_acc *acc);

void repro_acc_destroy(repro_acc *acc);

/* Shape queries. */
int32_t repro_acc_n_groups(const repro_acc *acc);
int32_t repro_acc_fold(const repro_acc *acc);
int32_t repro_acc_dtype(const repro_acc *acc);

/* ------------------------------------------------------------------------
 * Multi-GPU exchange (one process per GPU; the caller runs the collectives,
 * e.g. NCCL through torch.distributed).  Integer-only, so the result does
 * not depend on the collective's reduction order:
 *   1. repro_acc_top_levels(acc, k)          k: int32[n_groups] device
 *   2. all-reduce MAX over ranks on k
 *   3. repro_acc_window_export(acc, k, limbs) limbs: int64[n_groups*fold*2]
 *      (the group's level sums realigned to the global top k[g] -- the
 *      paper's level demotion, PAPER.md:660-665 -- as carry-split limbs
 *      lo in [0, 2^32), hi = floor(T / 2^32))
 *   4. all-reduce (or reduce-scatter by group range) SUM on limbs
 *   5. repro_acc_window_import(acc, k, limbs) (canonicalises, Alg. 1
 *      lines 17-21)
 * The result is bit-identical to depositing every rank's rows into one
 * handle.
 * ---------------------------------------------------------------------- */
int repro_acc_top_levels(const repro_acc *acc, int32_t *k_out);
int repro_acc_window_export(const repro_acc *acc, const int32_t *k_global,
                            int64_t *limbs_out);
int repro_acc_window_import(repro_acc *acc, const int32_t *k_global,
                            const int64_t *limbs);
/* Range form of window_import for a reduce-scatter by contiguous group
 * range: groups [g0, g0 + count) of the handle take the given limbs
 * (int64[count*fold*2]); k_global is int32[count] for that range. */
int repro_acc_window_import_range(repro_acc *acc, int32_t g0, int32_t count,
                                  const int32_t *k_global,
                                  const int64_t *limbs);

/* ------------------------------------------------------------------------
 * Non-reproducible baseline on the same GPU (BASELINE.json north_star):
 * out[g] = atomicAdd-accumulated sum in the value dtype (or in binary64 when
 * accumulate_f64 != 0 and dtype is F32).  variant 0: one global atomicAdd
 * per row; variant 1: shared-memory privatised table per block (compare-
 * and-swap on sm_100a) flushed with global atomics; variant 2 (n_groups <=
 * 16): per-thread register partials, one global atomic per group per warp;
 * variant 3: warp aggregation of equal keys (match.any), one global atomic
 * per distinct key per warp; variant 4: heavy hitters privatised (the keys
 * holding >= 1/2048 of 8192 sampled rows, at most 256, summed per warp in
 * shared memory and flushed once per block; the other rows by global
 * atomicAdd).  out is zeroed inside.  Stream-ordered,
 * non-blocking; returns REPRO_EINVAL for bad arguments or when the variant
 * does not apply (1: shared memory too small, 2: n_groups > 16).
 * ---------------------------------------------------------------------- */
int repro_baseline_atomic_sum(const int32_t *keys, const void *vals, int64_t n,
                              int32_t n_groups, int32_t dtype, int32_t variant,
                              int32_t accumulate_f64, void *out, void *stream);

/* Measurement support, not part of the method: the FP side of the roofline of
 * SURVEY.md 8(d) ("the deposit FLOPs at the vector FP64/FP32 peak").  Runs
 * independent chains of correctly rounded adds (__dadd_rn / __fadd_rn) of the
 * value type `dtype` on every SM and writes the measured adds per second of
 * the whole GPU (best of three launches) to *adds_per_s (host pointer).  The
 * digit cascade costs 3K - 2 adds per value (Alg. 1 lines 10-16,
 * PAPER.md:666-672).  Blocking (synchronises `stream`); EINVAL for an unknown
 * dtype or a null pointer, ECUDA on a CUDA error. */
int repro_measure_fp_add_rate(int32_t dtype, double *adds_per_s, void *stream);

/* ------------------------------------------------------------------------
 * Introspection for tests and the benchmark.
 * ---------------------------------------------------------------------- */
/* Number of kernels the last call on this host thread enqueued. */
int32_t repro_last_launch_count(void);
/* Path the last GroupBy call on this host thread took: 0 = on-chip tables,
 * 1 = radix-partitioned, 2 = fused multi-column on-chip pass, 3 = multi-column
 * call run one column at a time, -1 = none. */
int32_t repro_last_path(void);
/* Largest n_groups the on-chip path handles for (fold, dtype). */
int32_t repro_onchip_max_groups(int32_t fold, int32_t dtype);
/* Largest n_groups the two-pass sweep (partitioned path 1) handles. */
int32_t repro_sweep_max_groups(int32_t fold, int32_t dtype);
/* Force a path for testing: -1 auto (default), 0 on-chip, 1 partitioned
 * (the two-pass sweep where its 256 partitions suffice, else segmented radix
 * passes), 2 partitioned by segmented radix passes.  repro_last_path reports
 * the same numbers.  Never changes result bits. */
void repro_set_path_override(int32_t path);

/* Choose the on-chip accumulate kernel for testing: 0 auto (default: the
 * lean per-warp kernel for <= 16 groups single-column / <= 4 groups
 * multi-column, the keyless register kernel for repro_sum / repro_dot, else
 * the register-fed counter-table kernel k_table), 1 the per-row
 * shared-atomic kernel fed by a TMA ring, 2 k_table, 3 the per-row
 * shared-atomic kernel with register loads (no TMA).  Never changes result
 * bits. */
void repro_set_kernel_variant(int32_t variant);

/* Routed one-pass kernel of the partitioned path (k_route.cu), opt-in:
 * 1 on (used whenever the groups fit the SMs' shared-memory tables, about 1M
 * binary64 K=3 groups on 148 SMs), 0 off (default: the two-pass sweep runs;
 * the routed kernel measured slower on B200).  Rows move to the SM that owns their group through small L2
 * ring buffers (PartitionAndAggregate, with the partitions
 * streamed instead of materialised).  Never changes result bits. */
void repro_set_route_mode(int32_t mode);

/* Per-kernel device timing (benchmark aid).  While enabled, every kernel the
 * library enqueues from this host thread is bracketed by a CUDA event pair
 * recorded on the launching stream. */
void repro_timing_enable(int32_t on);
/* Synchronises on the recorded events and returns, for up to `max` distinct
 * kernels, their names (static strings), launch counts and summed device
 * milliseconds; clears the records.  Returns the number of kernels. */
int32_t repro_timing_collect(const char **names, int32_t *counts, double *total_ms, int32_t max);

#ifdef __cplusplus
}
#endif

#endif /* REPRO_GROUPBY_H */
