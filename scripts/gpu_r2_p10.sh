#!/bin/bash
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  echo "head: $(timeout 300 python scripts/variants/headpkg/sweep_head.py --nobase --groups 1024,4096 2>&1 | tail -2 | cut -c1-60 | tr '\n' ' ')"
  for v in x0p0 x1p1 x1p0; do
    echo "$v: $(REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 300 python scripts/sweep.py --nobase --groups 1024,4096 2>&1 | tail -2 | cut -c1-60 | tr '\n' ' ')"
  done
done
for v in x0p0 x1p1; do
  echo "$v zipf: $(REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 300 python scripts/sweep.py --nobase --skew --groups 1024,4096 2>&1 | tail -2 | cut -c1-60 | tr '\n' ' ')"
done
