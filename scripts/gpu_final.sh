cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/final/pytest_gpu.txt 2>&1; tail -3 gpurun_out/final/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1; tail -2 gpurun_out/final/smoke.txt
bash scripts/gpu_profiles.sh > /dev/null 2>&1
ls gpurun_out/prof | wc -l
