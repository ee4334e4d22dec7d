#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/swt
timeout 1500 python -m pytest tests/test_gpu_band.py tests/test_gpu_full_size.py tests/test_gpu_parity.py tests/test_gpu_sparse.py tests/test_gpu_edge.py tests/test_gpu_split.py tests/test_gpu_tune.py -x -q -p no:cacheprovider > gpurun_out/swt/t.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/swt/t.txt
