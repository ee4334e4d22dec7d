cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/variants.log
for v in scripts/variants/lib_*.so; do
  echo "== $v" >> gpurun_out/variants.log
  REPRO_B200_LIB=$PWD/$v timeout 300 python scripts/sweep.py --variant 1 --groups 16,256,1024,2048 >> gpurun_out/variants.log 2>&1
done
