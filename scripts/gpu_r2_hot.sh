#!/bin/bash
# hot-pass compaction rewrite: parity (band + route + full-size + edge) and timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/hot
timeout 1200 python -m pytest tests/test_gpu_band.py tests/test_gpu_full_size.py tests/test_gpu_edge.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/hot/t.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/hot/t.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e"
for c in "--config 3" "--config 2 --n-groups 16384" "--config 2 --n-groups 65536"; do
  timeout 300 $B $c > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c', round(d['ms_per_step'],3), d['parity']['vs_oracle'], {k: round(v,3) for k,v in d['per_kernel_ms'].items()})" || tail -3 /tmp/b.err
done
