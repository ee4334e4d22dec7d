cd $GRAFT_REPO_ROOT
O=gpurun_out/prof
mkdir -p $O
for c in 1 4; do
  extra=""; [ $c = 4 ] && extra="--rows 268435456"
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity $extra"
  $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c$c.csv $CMD > /dev/null 2>&1
done
