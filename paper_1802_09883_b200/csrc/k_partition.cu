// k_partition.cu -- radix-partitioned (high-cardinality) path: placeholder
// until the partition kernels land; the on-chip path covers n_groups up to
// repro_onchip_max_groups().
#include "internal.h"

namespace repro {

int partition_max_groups(int, int) { return 0; }
size_t partition_workspace_bytes(int64_t, int32_t, int, int) { return 0; }
int launch_partitioned(int, int, const int32_t *, const void *, int64_t, int32_t, void *, size_t, int, int32_t *,
                       int64_t *, int64_t *, void *, uint32_t *, cudaStream_t, int *) {
    return -1;
}

}  // namespace repro
