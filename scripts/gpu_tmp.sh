cd $GRAFT_REPO_ROOT
python scripts/check_variants.py 2>&1 | cut -c1-220
for v in w7; do echo $v; REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so python scripts/stress_variant.py 4194304 1024; done
NOCHECK=1 GROUPS_LIST=16,256,1024,2048 bash scripts/gpu_variants.sh; cat gpurun_out/variants.log | cut -c1-250
