// k_onchip.cu -- on-chip (low-cardinality) accumulate kernel.
//
// Hot path rows a1-a4/a6 of SURVEY.md section 8: stream <key, value> rows,
// compute each row's window top k* and its K integer digits (common.cuh),
// and add the digits into a per-block table of the group states held in
// shared memory (HashAggregation with identity hashing, PAPER.md:867-873,
// 1264).  Alg. 1's level check becomes an integer max:
// per tile of rows, every row raises its group's `ktop_next` (shared atomicMax)
// and, after one barrier, groups whose top moved shift their level sums down
// (the paper's demotion) before any digit of the tile is added.
//
// Digits are added with native 32-bit shared atomics (64-bit shared atomics
// are CAS loops on sm_100a): binary64 digits (|d| <= 2^39) are split into a
// 20-bit unsigned low limb and a signed high limb, binary32 digits fit one
// int32.  (MATCH.ANY costs ~64 cycles per warp on sm_100a and REDUX with a
// divergent mask compiles to a serial loop, so there is no general warp
// aggregation; only an all-lanes-same-group warp reduces first.)  Limb counters are folded into
// int64 level sums before they can overflow (Alg. 1's carry propagation,
// PAPER.md:673-679, deferred as in Alg. 2's NB blocking).
//
// At the end each block adds its int64 level sums into a global table indexed
// by ABSOLUTE lattice level (slot j + K - 1 for level j) with 64-bit global
// reductions, and raises the group's global top with atomicMax.  Because a
// row's digit at level j does not depend on which window it was computed in
// (digits above k* are zero), this table is exact whatever the block
// windows were; the fold kernel reads the K slots under the global top.
#include "common.cuh"
#include "internal.h"
#include "onchip_core.cuh"
#include "onchip_launch.cuh"

#include <algorithm>
#include <cstdlib>


namespace repro {

template <int DT, int K>
int launch_onchip(const int32_t *keys, const void *vals, int64_t n, int32_t G, int32_t *kglob,
                  unsigned long long *slots, uint32_t *status, cudaStream_t st, int *launches) {
    const SrcSingle<DT> src{{(const typename Fmt<DT>::V *)vals}, G};
    return launch_onchip_src<DT, K, SrcSingle<DT>, true>(keys, src, n, G, kglob, slots, status, st, launches);
}

int atomic_max_groups(int K, int DT) {
    // largest G whose table (level sums in shared memory, G rounded to 4)
    // fits; the register-sum kernel covers G <= REG_GQ in less space
    const size_t cap = (size_t)device_props().smem_optin;
    const size_t cw = (size_t)K * (DT == 1 ? 2 : 1);
    const size_t per = 8 * K + 4 * cw + 8;  // onchip_table_bytes = GQ * per + 64
    return (int)(((cap - 64 - 127) / per) & ~(size_t)3);
}

// variant: 0 = auto (k_lean for <= 16 groups, else k_table), 1 = the
// per-row atomic kernel fed by the TMA ring (accumulate_range), 2 = k_table,
// 3 = the per-row atomic kernel with register loads.  The bits never depend
// on the variant.  Initialised from REPRO_ONCHIP_VARIANT, settable through
// the C-ABI.
static int g_variant = -1;
int onchip_variant() {
    if (g_variant < 0) {
        const char *e = getenv("REPRO_ONCHIP_VARIANT");
        g_variant = (e && e[0] == 'a') ? 1 : (e && e[0] == 't') ? 2 : (e && e[0] == 'r') ? 3 : 0;
    }
    return g_variant;
}
void set_onchip_variant(int v) { g_variant = (v >= 0 && v <= 3) ? v : 0; }

int onchip_max_groups(int K, int DT) {
    const int v = onchip_variant();
    if (v == 1 || v == 3) return atomic_max_groups(K, DT);
    return table_max_groups(K, DT);
}

int launch_onchip_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G,
                      int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                      int *launches) {
    // a handful of groups: per-warp lane-copy tables (k_lean.cu); 1 = not taken
    const int lr = launch_lean_single(DT, K, keys, vals, n, G, kglob, slots, status, st, launches);
    if (lr != 1) return lr;
    const int v = onchip_variant();
    if (v == 1 || v == 3) return launch_atomic_any(DT, K, keys, vals, n, G, kglob, slots, status, st, launches);
    return launch_table_any(DT, K, keys, vals, n, G, kglob, slots, status, st, launches);
}

int launch_atomic_any(int DT, int K, const int32_t *keys, const void *vals, int64_t n, int32_t G,
                      int32_t *kglob, unsigned long long *slots, uint32_t *status, cudaStream_t st,
                      int *launches) {
    if (G > atomic_max_groups(K, DT)) return -1;
#define ONCHIP_CASE(dt, k) \
    if (DT == dt && K == k) return launch_onchip<dt, k>(keys, vals, n, G, kglob, slots, status, st, launches);
    ONCHIP_CASE(1, 1) ONCHIP_CASE(1, 2) ONCHIP_CASE(1, 3) ONCHIP_CASE(1, 4)
    ONCHIP_CASE(0, 1) ONCHIP_CASE(0, 2) ONCHIP_CASE(0, 3) ONCHIP_CASE(0, 4)
#undef ONCHIP_CASE
    return -1;
}

}  // namespace repro
