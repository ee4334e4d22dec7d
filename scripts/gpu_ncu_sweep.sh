#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_split.py -q -x > gpurun_out/r2d_split.log 2>&1
tail -2 gpurun_out/r2d_split.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep" -c 2 -o gpurun_out/ncu_sweep -f python scripts/sweep.py --groups 1048576 --pm1 --n 268435456 --nobase > gpurun_out/ncu_sweep.log 2>&1
tail -3 gpurun_out/ncu_sweep.log
: > gpurun_out/tabpf.log
for v in scripts/variants/lib_pf*.so; do
  echo "== $v" >> gpurun_out/tabpf.log
  REPRO_B200_LIB=$PWD/$v timeout 300 python scripts/sweep.py --nobase --groups 1024,4096 >> gpurun_out/tabpf.log 2>&1
  REPRO_B200_LIB=$PWD/$v timeout 300 python scripts/sweep.py --nobase --groups 1024 --pm1 --n 268435456 >> gpurun_out/tabpf.log 2>&1
done
cat gpurun_out/tabpf.log
