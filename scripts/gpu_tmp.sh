cd $GRAFT_REPO_ROOT
for v in i8 i4 i16; do
for G in 65536 1048576; do
REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 900 python bench.py --config 2 --n-groups $G --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-atomic-baseline --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 $G $v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"
done
REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-atomic-baseline --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"
done
