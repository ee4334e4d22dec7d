cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tune.py tests/test_gpu_full_size.py -q -x 2>&1 | tail -2
for G in 262144 1048576 4194304; do timeout 600 python bench.py --config 2 --n-groups $G --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($G, round(d['ms_per_step'],3), d['parity']['vs_oracle'], round(d['step_roofline_frac'],3), round(d['baseline_atomic']['slowdown_repro_vs_atomic'],2), {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"; done
