#!/bin/bash
# round-2 closing evidence: GPU suite, smoke, default bench (all configs), reference arm, launch lists
# (config 1, config 2 at G = 2^20), ncu --set full of the sweep's scatter + accumulate at G = 2^16
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fin3
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin3/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin3/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin3/smoke.txt
timeout 1800 python bench.py > gpurun_out/fin3/bench.json 2> gpurun_out/fin3/bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/fin3/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/fin3/bench_ref.json 2> gpurun_out/fin3/bench_ref.err; echo "ref rc=$?"
Q="--no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin3/c1_launches.csv python bench.py --steps 2 --warmup 3 $Q > /dev/null 2>&1; echo "c1 launches rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin3/g20_launches.csv python bench.py --config 2 --n-groups 1048576 --steps 2 --warmup 3 $Q > /dev/null 2>&1; echo "g20 launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_cold|k_sweep_acc" -c 2 -o gpurun_out/fin3/g65k python bench.py --config 2 --n-groups 65536 --steps 1 --warmup 3 $Q > gpurun_out/fin3/ncu_g65k.log 2>&1; echo "g65k ncu rc=$?"
