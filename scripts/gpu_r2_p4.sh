#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2d
REPRO_B200_LIB=$PWD/scripts/variants/lib_dbg.so timeout 300 python scripts/dbg_modes.py 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -p no:cacheprovider > gpurun_out/r2d/tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2d/tests.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e --no-parity"
for c in "--config 1" "--config 2 --n-groups 4096" "--config 2 --n-groups 1024" "--config 3"; do
  timeout 600 $B $c > gpurun_out/r2d/b.json 2>gpurun_out/r2d/b.err
  python -c "import json; d=json.load(open('gpurun_out/r2d/b.json')); print('$c', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['per_kernel_ms'].items()})" || tail -3 gpurun_out/r2d/b.err
done
