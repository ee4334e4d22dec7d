cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -5
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['ms_per_step'], d['parity']['vs_oracle'], d['roofline']['frac'], {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"
