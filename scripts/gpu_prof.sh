# launch list (cold, serialised) + one full ncu capture of the dominant kernel
# of `bench.py` at its default config -> gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-parity ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 30 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-onchip} -s 2 -c 1 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
