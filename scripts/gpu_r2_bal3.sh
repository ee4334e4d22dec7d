#!/bin/bash
# parallel cost-balanced cuts, warp-match scatter ranks for P <= 8, fused radix offsets (sparse)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bal3
timeout 1200 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_band.py tests/test_gpu_full_size.py tests/test_gpu_parity.py tests/test_gpu_split.py tests/test_gpu_tune.py -q -p no:cacheprovider -x > gpurun_out/bal3/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bal3/pytest.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e --no-parity"
for c in "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576" "--config 3" "--config 2 --n-groups 16384" "--config 2 --n-groups 8192" "--config 2 --n-groups 262144"; do
  timeout 300 $B $c > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_kernel_ms'].items()})" || tail -3 /tmp/b.err
done
timeout 600 python -c "import json, torch, bench, paper_1802_09883_b200 as R; d=bench.run_sparse(R, torch, 5, 3); print('f1', d['ms_per_step'], d.get('parity'))"; echo "f1 rc=$?"
