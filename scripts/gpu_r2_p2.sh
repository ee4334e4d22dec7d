#!/bin/bash
# new scatter: parity + timings + ncu of the table kernels in band/uniform modes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_parity.py tests/test_gpu_split.py -x -q -p no:cacheprovider -k "band or partitioned or split or sweep" > gpurun_out/r2c/tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2c/tests.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e"
for c in "--config 3" "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576" "--config 1" "--config 2 --n-groups 4096"; do
  timeout 600 $B $c > gpurun_out/r2c/b.json 2>gpurun_out/r2c/b.err
  python -c "import json; d=json.load(open('gpurun_out/r2c/b.json')); print('$c', round(d['ms_per_step'],3), d['parity']['vs_oracle'], {k: round(v,3) for k,v in d['per_kernel_ms'].items()})" || tail -3 gpurun_out/r2c/b.err
done
N="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_table -s 3 -c 1 -o gpurun_out/r2c/c1 -f $N --config 1 > /dev/null 2>&1; echo "c1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_table -s 3 -c 1 -o gpurun_out/r2c/g4k -f $N --config 2 --n-groups 4096 > /dev/null 2>&1; echo "g4k rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_sw_" -s 6 -c 6 -o gpurun_out/r2c/c3 -f $N --config 3 > /dev/null 2>&1; echo "c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep_cold|k_sw_hist" -s 2 -c 2 -o gpurun_out/r2c/c2m -f $N --config 2 --n-groups 1048576 > /dev/null 2>&1; echo "c2m rc=$?"
