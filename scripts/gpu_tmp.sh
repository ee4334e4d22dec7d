cd $GRAFT_REPO_ROOT
python scripts/check_variants.py 2>&1 | cut -c1-220
for v in lane32; do echo $v; for g in 1 4 16 32; do REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so python scripts/stress_variant.py 4194304 $g; done; done
NOCHECK=1 GROUPS_LIST=1,4,16,32,64 bash scripts/gpu_variants.sh; cat gpurun_out/variants.log | cut -c1-250
