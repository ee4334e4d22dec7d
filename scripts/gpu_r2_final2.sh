#!/bin/bash
# round-2 final evidence: GPU suite, smoke, default bench (all configs), reference arm, config-1 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fin2
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin2/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin2/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin2/smoke.txt
timeout 1800 python bench.py > gpurun_out/fin2/bench.json 2> gpurun_out/fin2/bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/fin2/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/fin2/bench_ref.json 2> gpurun_out/fin2/bench_ref.err; echo "ref rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin2/c1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin2/c3_launches.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e > /dev/null 2>&1; echo "c3 launches rc=$?"
