cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/lean
CMD="python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --rows 268435456"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:lean -s 2 -c 1 -o gpurun_out/lean/full_c4 $CMD > gpurun_out/lean/ncu.log 2>&1
tail -3 gpurun_out/lean/ncu.log
