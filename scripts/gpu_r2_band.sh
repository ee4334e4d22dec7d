#!/bin/bash
# band-mode tables: parity + config-3 / sweep timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_band.py -x -q -p no:cacheprovider > gpurun_out/r2b/band.txt 2>&1; echo "band rc=$?"; tail -3 gpurun_out/r2b/band.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2b/all.txt 2>&1; echo "all rc=$?"; tail -3 gpurun_out/r2b/all.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e"
for c in "--config 3" "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576" "--config 1" "--config 2 --n-groups 4096"; do
  timeout 600 $B $c > gpurun_out/r2b/b.json 2>gpurun_out/r2b/b.err
  python -c "import json; d=json.load(open('gpurun_out/r2b/b.json')); print('$c', round(d['ms_per_step'],3), d['parity']['vs_oracle'], {k: round(v,3) for k,v in d['per_kernel_ms'].items()})" || tail -3 gpurun_out/r2b/b.err
done
