cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "partition or heavy" 2>&1 | tail -2
for v in s8 s12 s16; do
for G in 16384 262144; do
REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 900 python bench.py --config 2 --n-groups $G --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-atomic-baseline --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 $G $v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"
done
done
REPRO_B200_LIB=$PWD/scripts/variants/lib_s8.so timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-atomic-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['ms_per_step'],3), d['parity']['vs_oracle'], {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"
