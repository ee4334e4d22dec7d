cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tune.py -q -x -k "partition or tune or Tune" 2>&1 | tail -3
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['ms_per_step'], d['parity']['vs_oracle'], {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"
for G in 4096 262144 524288 1048576; do timeout 600 python bench.py --config 2 --n-groups $G --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-atomic-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($G, d['ms_per_step'], d['parity']['vs_oracle'], {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"; done
