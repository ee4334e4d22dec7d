#!/bin/bash
# A/B of k_table tuning variants on config 1 (2^27 rows, G=1024)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in base vlo0 qpt3; do
  REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"
done
done
