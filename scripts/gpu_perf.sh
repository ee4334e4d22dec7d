cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/sweep.py --variant 1 --groups 1,16,256,1024,2048,3000 > gpurun_out/sweep.log 2>&1
timeout 600 python scripts/sweep.py --variant 1 --dtype f32 --fold 2 --groups 1,1024,4096 >> gpurun_out/sweep.log 2>&1
export REPRO_ONCHIP_VARIANT=a
CMD="python bench.py --steps 3 --warmup 1 --rows 67108864 --no-e2e --no-cpu-baseline --no-atomic-baseline --no-parity"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:onchip -c 1 -o gpurun_out/prof_atomic4 $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
