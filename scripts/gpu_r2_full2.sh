#!/bin/bash
# full check: GPU suite, smoke, default bench (all configs), config-1 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2g
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2g/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2g/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2g/smoke.txt
timeout 1500 python bench.py > gpurun_out/r2g/bench.json 2> gpurun_out/r2g/bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r2g/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g/c1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
