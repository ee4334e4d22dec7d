#!/bin/bash
# A/B the k_table tuning variants (scripts/variants/lib_*.so): config-1 shape
# and a group-count sweep, fp64 K=3 and fp32 K=2
cd $GRAFT_REPO_ROOT
: > gpurun_out/tabvar.log
for v in scripts/variants/lib_*.so; do
  echo "== $v" >> gpurun_out/tabvar.log
  REPRO_B200_LIB=$PWD/$v timeout 300 python scripts/sweep.py --nobase --variant 2 --groups 64,1024,2048,4096,7000 >> gpurun_out/tabvar.log 2>&1
  REPRO_B200_LIB=$PWD/$v timeout 300 python scripts/sweep.py --nobase --variant 2 --dtype f32 --fold 2 --groups 1024,8192,16000 >> gpurun_out/tabvar.log 2>&1
done
