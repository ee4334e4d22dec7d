cd $GRAFT_REPO_ROOT
for v in o64_7 o64_8 o64_10; do
  echo "== $v"
  export REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so
  for G in 262144 1048576; do
    timeout 600 python bench.py --config 2 --n-groups $G --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-atomic-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($G, round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['per_kernel_ms'].items()})"
  done
done
