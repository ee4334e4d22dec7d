#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "partitioned or carry or edge_rows" > gpurun_out/r2g_tests.log 2>&1
tail -2 gpurun_out/r2g_tests.log
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs > gpurun_out/r2g_c3.json 2> gpurun_out/r2g_c3.err
python -c "import json; d=json.load(open('gpurun_out/r2g_c3.json')); print(d['ms_per_step'], d['per_kernel_ms'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sw_hist|k_sweep_cold|k_sweep_acc" -c 3 -o gpurun_out/ncu_sw3 -f python scripts/sweep.py --groups 1048576 --pm1 --n 268435456 --nobase > gpurun_out/ncu_sw3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep_hot" -c 1 -o gpurun_out/ncu_swhot -f python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e > gpurun_out/ncu_swhot.log 2>&1
tail -2 gpurun_out/ncu_sw3.log gpurun_out/ncu_swhot.log
