cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -x -k "lean or variant or few or config4 or moments or random" 2>&1 | tail -2
for G in 1 16; do timeout 600 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-atomic-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($G, round(d['ms_per_step'],4), d['parity']['vs_oracle'], round(d['roofline']['frac'],3), d['roofline']['kernel'])"; done
