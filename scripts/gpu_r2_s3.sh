#!/bin/bash
# session-3 state check: GPU suite, smoke, per-config timings with kernel breakdown
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s3/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s3/smoke.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e"
for c in "--config 1" "--config 3" "--config 2 --n-groups 4096" "--config 2 --n-groups 16384" "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576" "--config 2 --n-groups 16777216"; do
  timeout 600 $B $c > gpurun_out/s3/b.json 2>gpurun_out/s3/b.err
  python -c "import json; d=json.load(open('gpurun_out/s3/b.json')); print('$c', round(d['ms_per_step'],3), d['parity']['vs_oracle'], {k: round(v,3) for k,v in d['per_kernel_ms'].items()})" || tail -3 gpurun_out/s3/b.err
done
