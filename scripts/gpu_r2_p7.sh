#!/bin/bash
# same-box A/B: HEAD (round-2 start) vs current k_table variants, config-1 shape (sweep.py timing)
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  echo "head: $(timeout 300 python scripts/variants/headpkg/sweep_head.py --nobase --groups 1024 2>&1 | tail -1)"
  for v in tb0 tb s4k; do
    echo "$v: $(REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 300 python scripts/sweep.py --nobase --groups 1024 2>&1 | tail -1)"
  done
done
