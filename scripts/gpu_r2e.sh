#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_split.py -q -x -k "partitioned or split or carry or edge_rows" > gpurun_out/r2e_tests.log 2>&1
tail -2 gpurun_out/r2e_tests.log
timeout 300 python scripts/sweep.py --groups 7000,16384,65536,262144,1048576 --pm1 --n 268435456 --nobase > gpurun_out/r2e_sweep64.log 2>&1
timeout 300 python scripts/sweep.py --groups 16384,262144,1048576 --dtype f32 --fold 2 --n 268435456 --nobase > gpurun_out/r2e_sweep32.log 2>&1
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline > gpurun_out/r2e_c3.json 2> gpurun_out/r2e_c3.err
cat gpurun_out/r2e_sweep64.log gpurun_out/r2e_sweep32.log
python -c "import json; d=json.load(open('gpurun_out/r2e_c3.json')); print(d['ms_per_step'], d['per_kernel_ms'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep" -c 3 -o gpurun_out/ncu_sweep2 -f python scripts/sweep.py --groups 1048576 --pm1 --n 268435456 --nobase > gpurun_out/ncu_sweep2.log 2>&1
