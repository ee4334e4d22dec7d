cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/final2/pytest_gpu.txt 2>&1; tail -2 gpurun_out/final2/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final2/smoke.txt 2>&1; tail -2 gpurun_out/final2/smoke.txt
timeout 900 python bench.py > gpurun_out/final2/bench_c1.json 2> gpurun_out/final2/bench_c1.err; head -c 300 gpurun_out/final2/bench_c1.json
