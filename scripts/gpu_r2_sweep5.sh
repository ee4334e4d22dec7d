#!/bin/bash
# round-2 group-count sweep of config 2 (2^28 rows fp64 U[-1,1), K=3): one bench line per G with parity against
# the oracle, the fastest atomicAdd comparator and per-kernel times (the paper's group-count figure, PAPER.md 1630-1643)
cd $GRAFT_REPO_ROOT
O=gpurun_out/sweep5; mkdir -p $O
: > $O/sweep_config2.jsonl
for G in 1 4 16 64 256 1024 2048 4096 6144 8192 16384 65536 262144 1048576 4194304 16777216; do
  timeout 400 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-configs --no-e2e --no-cpu-baseline >> $O/sweep_config2.jsonl 2>> $O/sweep.err; echo "G=$G rc=$?"
done
