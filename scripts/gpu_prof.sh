cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 1 --rows 16777216 --no-e2e --no-cpu-baseline --no-atomic-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:onchip -c 1 -o gpurun_out/prof_sorted $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
