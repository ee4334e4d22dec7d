#!/bin/bash
# A/B of k_table tuning variants on the config-1 shape and G=1024/4096 (2^28 rows, U[-1,1))
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2v
: > gpurun_out/r2v/var.log
for rep in 1 2; do
for v in scripts/variants/lib_*.so; do
  echo "== $v" >> gpurun_out/r2v/var.log
  REPRO_B200_LIB=$PWD/$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config1', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))" >> gpurun_out/r2v/var.log 2>&1
  REPRO_B200_LIB=$PWD/$v timeout 300 python scripts/sweep.py --nobase --groups 1024,4096 --pm1 --n 268435456 >> gpurun_out/r2v/var.log 2>&1
done
done
cat gpurun_out/r2v/var.log
