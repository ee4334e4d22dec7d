#!/bin/bash
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  echo "head: $(timeout 300 python scripts/variants/headpkg/sweep_head.py --nobase --groups 1024,4096 2>&1 | tail -2 | tr '\n' ' ')"
  for v in pair pair0; do
    echo "$v: $(REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 300 python scripts/sweep.py --nobase --groups 1024,4096 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
REPRO_B200_LIB=$PWD/scripts/variants/lib_pair.so timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -p no:cacheprovider > gpurun_out/p9tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/p9tests.txt
