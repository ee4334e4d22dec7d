#!/bin/bash
# one-block-per-SM k_table (2048 < G <= 6.3K): 512 vs 384 threads, 1 vs 2 quads per thread
cd $GRAFT_REPO_ROOT
for v in main t384q1 t384q2; do
  L=""; [ $v != main ] && L="REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so"
  env $L timeout 300 python scripts/sweep.py --nobase --groups 3000,4096,6000 --n 134217728 2>&1 | sed "s/^/$v /" | cut -c1-100
  env $L timeout 300 python scripts/sweep.py --nobase --pm1 --groups 4096 --n 268435456 2>&1 | sed "s/^/$v pm1 /" | cut -c1-100
done
