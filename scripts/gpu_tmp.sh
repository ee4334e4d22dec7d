cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/lean16
CMD="python bench.py --config 2 --n-groups 16 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-atomic-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:lean -s 2 -c 1 -o gpurun_out/lean16/full $CMD > gpurun_out/lean16/ncu.log 2>&1
tail -1 gpurun_out/lean16/ncu.log
