cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -4
timeout 600 python bench.py --steps 50 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['parity']['vs_oracle'], round(d['roofline']['frac'],3), d['roofline']['kernel'], d['baseline_atomic']['slowdown_repro_vs_atomic'])"
for G in 64 256 1024; do timeout 600 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($G, d['ms_per_step'], d['parity']['vs_oracle'], round(d['roofline']['frac'],3), d['roofline']['kernel'])"; done
