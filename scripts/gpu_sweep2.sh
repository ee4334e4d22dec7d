cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python scripts/sweep.py --n 268435456 --pm1 > gpurun_out/sweep_cfg2.log 2>&1
timeout 600 python scripts/sweep.py --n 268435456 --dtype f32 --fold 2 --skew --groups 1048576 > gpurun_out/sweep_cfg3.log 2>&1
