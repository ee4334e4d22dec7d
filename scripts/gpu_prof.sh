cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export REPRO_ONCHIP_VARIANT=a
CMD="python bench.py --steps 3 --warmup 1 --rows 67108864 --no-e2e --no-cpu-baseline --no-atomic-baseline --no-parity"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:onchip -c 1 -o gpurun_out/prof_atomic3 $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
