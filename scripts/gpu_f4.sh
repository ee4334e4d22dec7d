# f4 evidence: GPU parity of the keyless SUM/dot, bench lines, launch list and
# a full ncu capture of k_rsum -> gpurun_out/f4/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/f4
O=gpurun_out/f4
timeout 900 python -m pytest tests/test_gpu_array.py -q -x > $O/tests.txt 2>&1; tail -2 $O/tests.txt
for c in 5 6; do
  timeout 900 python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err; cat $O/bench_c$c.json | head -c 1500; echo
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-parity"
  $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c$c.csv $CMD > /dev/null 2>&1
  $CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rsum -s 2 -c 1 -o $O/full_c$c $CMD > /dev/null 2>&1
done
ls -la $O
