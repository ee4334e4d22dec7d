cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_array.py -q -x 2>&1 | tail -3
timeout 300 python scripts/array_perf.py
