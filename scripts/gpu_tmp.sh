cd $GRAFT_REPO_ROOT
GROUPS_LIST=16,256,1024,2048,4096 bash scripts/gpu_variants.sh
cat gpurun_out/variants.log
