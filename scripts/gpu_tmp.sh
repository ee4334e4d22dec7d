cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in r7 r8; do
REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 900 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-parity --no-atomic-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 $v', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
done
done
for v in r7 r8; do
for G in 32 4096; do
REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so timeout 900 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-atomic-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 $G $v', round(d['ms_per_step'],4))"
done
done
