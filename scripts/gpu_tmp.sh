cd $GRAFT_REPO_ROOT
O=gpurun_out/prof2; mkdir -p $O
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
for c in 1 3 4; do
  extra=""; [ $c = 4 ] && extra="--rows 268435456"
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity $extra"
  $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c$c.csv $CMD > /dev/null 2>&1
done
ls -la $O
