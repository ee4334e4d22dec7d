#!/bin/bash
# replicated-read form enabled by default for 2-partition plans: A/B on other formats, then the whole GPU suite,
# smoke and the default bench at this build
cd $GRAFT_REPO_ROOT
O=gpurun_out/rep2; mkdir -p $O
for M in 0 2 3; do
  echo "== REPRO_SWEEP_REP_MAXP=$M" >> $O/ab.txt
  REPRO_SWEEP_REP_MAXP=$M timeout 300 python scripts/sweep.py --n 268435456 --pm1 --dtype f32 --fold 2 --nobase --groups 12288,16384,20000,24576 >> $O/ab.txt 2>&1
  REPRO_SWEEP_REP_MAXP=$M timeout 300 python scripts/sweep.py --n 268435456 --pm1 --dtype f64 --fold 2 --nobase --groups 8192,12288,16384,24576 >> $O/ab.txt 2>&1
  REPRO_SWEEP_REP_MAXP=$M timeout 300 python scripts/sweep.py --n 268435456 --pm1 --dtype f64 --fold 3 --nobase --groups 6500,7000,8192 >> $O/ab.txt 2>&1
done
cut -c1-110 $O/ab.txt
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout 1800 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 300 $O/bench.err
timeout 300 python bench.py --config 2 --n-groups 8192 --steps 20 --warmup 3 --no-configs --no-e2e --no-cpu-baseline > $O/g8192.json 2>> $O/bench.err; echo "g8192 rc=$?"
Q="--no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/g8192_launches.csv python bench.py --config 2 --n-groups 8192 --steps 2 --warmup 3 $Q > /dev/null 2>&1; echo "g8192 launches rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:k_sweep_hot -s 3 -c 1 -f -o $O/g8192_rep python bench.py --config 2 --n-groups 8192 --steps 1 --warmup 3 $Q > $O/ncu_g8192.log 2>&1; echo "g8192 ncu rc=$?"
python scripts/ncu_summary.py $O/g8192_rep.ncu-rep > $O/g8192_rep.txt 2>&1; rm -f $O/g8192_rep.ncu-rep
