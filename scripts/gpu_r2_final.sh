#!/bin/bash
# round-2 evidence: default bench (all configs), reference arm, smoke, config-1 launch list + ncu full of the top kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fin
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin/smoke.txt
timeout 1800 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/fin/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err; echo "ref rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/c1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_table -c 1 -o gpurun_out/fin/c1_table python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e > gpurun_out/fin/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
