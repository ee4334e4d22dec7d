#!/bin/bash
# replicated-read form of the sweep (plans of 2-4 partitions): parity tests, then A/B timing against the scatter form
cd $GRAFT_REPO_ROOT
O=gpurun_out/rep; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_replicated.py -q -p no:cacheprovider -x > $O/pytest_rep.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_rep.txt
for M in 0 4; do
  for G in 8192 12288 16384; do
    REPRO_SWEEP_REP_MAXP=$M timeout 300 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-configs --no-e2e --no-cpu-baseline >> $O/rep_maxp$M.jsonl 2>> $O/rep.err; echo "M=$M G=$G rc=$?"
  done
done
for M in 0 4; do python scripts/bench_table.py $O/rep_maxp$M.jsonl; done
