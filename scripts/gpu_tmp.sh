cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "partition or heavy" 2>&1 | tail -2
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-atomic-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['ms_per_step'], d['parity']['vs_oracle'], {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"
