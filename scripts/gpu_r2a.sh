#!/bin/bash
# round-2 check: parity of the new k_table path + old-kernel fold fix, and a quick perf A/B
python scripts/dbg_fold.py > gpurun_out/dbg_fold2.log 2>&1
python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -q -x > gpurun_out/r2a_tests.log 2>&1
for v in a t; do
  for cfg in "--config 1" "--config 2 --n-groups 64" "--config 2 --n-groups 1024" "--config 2 --n-groups 4096"; do
    REPRO_ONCHIP_VARIANT=$v python bench.py $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-parity >> gpurun_out/r2a_bench_$v.jsonl 2>>gpurun_out/r2a_bench.err
  done
done
tail -3 gpurun_out/r2a_tests.log
