cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host" 2>&1 | tail -1
timeout 900 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
