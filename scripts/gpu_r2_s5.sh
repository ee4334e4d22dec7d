#!/bin/bash
# session-5 closing evidence at HEAD: GPU suite, smoke, default bench (all configs), reference arm,
# launch lists (config 1, config 3, config 2 at G = 2^16), ncu --set full of k_table (config 1) and of the
# sweep's scatter + accumulate at G = 2^16 (after the static-range accumulate)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5; mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout 1800 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 300 $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
Q="--no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c1_launches.csv python bench.py --steps 2 --warmup 3 $Q > /dev/null 2>&1; echo "c1 launches rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c3_launches.csv python bench.py --config 3 --steps 2 --warmup 3 $Q > /dev/null 2>&1; echo "c3 launches rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/g16_launches.csv python bench.py --config 2 --n-groups 65536 --steps 2 --warmup 3 $Q > /dev/null 2>&1; echo "g16 launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_table -s 3 -c 1 -f -o $O/c1 python bench.py --steps 1 --warmup 3 $Q > $O/ncu_c1.log 2>&1; echo "c1 ncu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_cold|k_sweep_acc" -c 2 -f -o $O/g65k python bench.py --config 2 --n-groups 65536 --steps 1 --warmup 3 $Q > $O/ncu_g65k.log 2>&1; echo "g65k ncu rc=$?"
ls -la $O
