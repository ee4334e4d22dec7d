#!/bin/bash
# session-4 re-entry check: GPU suite, smoke, default bench at HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s4
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/s4/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4/smoke.txt
timeout 1800 python bench.py > gpurun_out/s4/bench.json 2> gpurun_out/s4/bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/s4/bench.err
