cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/variants.log
[ -z "$NOCHECK" ] && python scripts/check_variants.py >> gpurun_out/variants.log 2>&1
for v in scripts/variants/lib_*.so; do
  echo "== $v" >> gpurun_out/variants.log
  REPRO_B200_LIB=$PWD/$v timeout 300 python scripts/sweep.py --nobase --variant 1 --groups ${GROUPS_LIST:-16,256,1024,2048} >> gpurun_out/variants.log 2>&1
  REPRO_B200_LIB=$PWD/$v timeout 300 python scripts/sweep.py --nobase --pm1 --variant 1 --groups 1024 >> gpurun_out/variants.log 2>&1
done
