cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "partitioned" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python scripts/sweep.py --n 268435456 --pm1 --groups 4096,65536,1048576,16777216 > gpurun_out/sweep_cfg2.log 2>&1
timeout 600 python scripts/sweep.py --n 268435456 --dtype f32 --fold 2 --skew --groups 1048576 > gpurun_out/sweep_cfg3.log 2>&1
