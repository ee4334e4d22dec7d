#!/bin/bash
# round-2: parity of k_table + sweep, then perf of both, then the full bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -q -x > gpurun_out/r2b_tests.log 2>&1
tail -3 gpurun_out/r2b_tests.log
timeout 300 python scripts/sweep.py --groups 1024,4096,7000,16384,65536,262144,1048576 --pm1 --n 268435456 > gpurun_out/r2b_sweep64.log 2>&1
timeout 300 python scripts/sweep.py --groups 8192,16384,65536,262144,1048576 --dtype f32 --fold 2 --n 268435456 > gpurun_out/r2b_sweep32.log 2>&1
cat gpurun_out/r2b_sweep64.log gpurun_out/r2b_sweep32.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
tail -3 gpurun_out/r2b_bench.err
