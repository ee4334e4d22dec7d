#!/bin/bash
# k_table defaults (QPT 2 + OBS2) vs the old ones over group counts; then the GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tab
for v in main old q512x2; do
  L=""; [ $v != main ] && L="REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so"
  env $L timeout 300 python scripts/sweep.py --nobase --groups 24,64,300,1024,2048,3000,4096,6000 --n 134217728 2>&1 | sed "s/^/$v /" | cut -c1-110
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tab/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tab/pytest_gpu.txt
