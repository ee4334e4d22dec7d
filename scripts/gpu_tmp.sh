cd $GRAFT_REPO_ROOT
python scripts/check_variants.py 2>&1 | cut -c1-200
NOCHECK=1 GROUPS_LIST=16,256,1024 bash scripts/gpu_variants.sh; cat gpurun_out/variants.log | cut -c1-120
for v in zs1 zs0; do export REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so; timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c4', d['ms_per_step'])"; done
