#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_parity.py -q -x -k "split or partitioned or merge" > gpurun_out/r2c_tests.log 2>&1
tail -3 gpurun_out/r2c_tests.log
timeout 300 python scripts/sweep.py --groups 7000,16384,65536,262144,1048576 --pm1 --n 268435456 > gpurun_out/r2c_sweep64.log 2>&1
timeout 300 python scripts/sweep.py --groups 16384,262144,1048576 --dtype f32 --fold 2 --n 268435456 > gpurun_out/r2c_sweep32.log 2>&1
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/r2c_c3.json 2> gpurun_out/r2c_c3.err
cat gpurun_out/r2c_sweep64.log gpurun_out/r2c_sweep32.log
python -c "import json; d=json.load(open('gpurun_out/r2c_c3.json')); print(d['ms_per_step'], d['per_kernel_ms'])"
