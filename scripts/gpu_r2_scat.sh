#!/bin/bash
# scatter with staged destinations: parity of every sweep user + timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/scat
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e --no-parity"
for c in "--config 3" "--config 2 --n-groups 16384" "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576"; do
  timeout 300 $B $c > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_kernel_ms'].items()})" || tail -3 /tmp/b.err
done
timeout 1500 python -m pytest tests/test_gpu_band.py tests/test_gpu_full_size.py tests/test_gpu_parity.py tests/test_gpu_sparse.py tests/test_gpu_edge.py tests/test_gpu_split.py tests/test_gpu_tune.py -x -q -p no:cacheprovider > gpurun_out/scat/t.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/scat/t.txt
