#!/bin/bash
# per-lane sink columns: full GPU suite + timings of the table-based configs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sink
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e --no-parity"
for c in "--config 3" "--config 1" "--config 2 --n-groups 4096" "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576"; do
  timeout 300 $B $c > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_kernel_ms'].items()})" || tail -3 /tmp/b.err
done
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/sink/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/sink/pytest_gpu.txt
