cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -x 2>&1 | tail -4
for G in 1 4 16; do timeout 600 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($G, d['ms_per_step'], d['parity']['vs_oracle'], round(d['roofline']['frac'],3), d['roofline']['kernel'])"; done
timeout 600 python bench.py --config 0 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c0', d['ms_per_step'], d['parity']['vs_oracle'], d['roofline']['kernel'])"
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['ms_per_step'], d['parity']['vs_oracle'], round(d['roofline']['frac'],3))"
