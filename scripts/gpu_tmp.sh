cd $GRAFT_REPO_ROOT
for v in m2 m3 m4; do
  export REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so
  echo "== $v"; timeout 900 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -1
  timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['parity']['vs_oracle'])"
done
