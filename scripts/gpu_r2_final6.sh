#!/bin/bash
# closing evidence with the replicated-read form on for plans of 2-3 partitions: GPU suite, smoke, default bench,
# reference arm, config-2 sweep over the former cliff, launch list at G = 8192
cd $GRAFT_REPO_ROOT
O=gpurun_out/fin6; mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout 1800 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 300 $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
for G in 6144 7000 8192 10000 12288 16384; do
  timeout 400 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-configs --no-e2e --no-cpu-baseline >> $O/sweep_cliff.jsonl 2>> $O/sweep.err; echo "G=$G rc=$?"
done
Q="--no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/g8192_launches.csv python bench.py --config 2 --n-groups 8192 --steps 2 --warmup 3 $Q > /dev/null 2>&1; echo "g8192 launches rc=$?"
