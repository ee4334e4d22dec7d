#!/bin/bash
# Round-2 full check: GPU suite, smoke, default bench (all configs), launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
t0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/r2/pytest_gpu.txt 2>&1; echo "pytest rc=$? $(( $(date +%s)-t0 ))s"
tail -3 gpurun_out/r2/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2/smoke.txt
t0=$(date +%s)
timeout 1500 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$? $(( $(date +%s)-t0 ))s"
tail -c 600 gpurun_out/r2/bench.err
