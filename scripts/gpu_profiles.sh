# Round-end evidence: bench lines for configs 1-4 (+ config 2 sweep), launch
# lists and full ncu captures of the dominant kernels -> gpurun_out/prof/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
O=gpurun_out/prof
timeout 900 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $O/bench_ref_c1.json 2> $O/bench_ref_c1.err
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config 5 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --config 6 > $O/bench_c6.json 2> $O/bench_c6.err
: > $O/sweep_c2.jsonl
for G in 1 4 16 64 256 1024 4096 16384 65536 262144 1048576 4194304 16777216; do
  timeout 600 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/sweep_c2.jsonl 2>> $O/sweep_c2.err
done
for c in 1 3 4; do
  extra=""; [ $c = 4 ] && extra="--rows 268435456"
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity $extra"
  $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c$c.csv $CMD > /dev/null 2>&1
done
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-parity"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:onchip -s 2 -c 1 -o $O/full_c1 $CMD > /dev/null 2>&1
CMD="python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --rows 268435456"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:lean -s 2 -c 1 -o $O/full_c4 $CMD > /dev/null 2>&1
CMD="python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-atomic-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"seg_scatter|part_accumulate" -s 2 -c 2 -o $O/full_c3 $CMD > /dev/null 2>&1
ls -la $O
