cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_synth.py -q 2>&1 | tail -2
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "rc=$?"; tail -3 gpurun_out/bench_c4.err
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "rc=$?"; tail -3 gpurun_out/bench_c1.err
cat gpurun_out/bench_c4.json gpurun_out/bench_c1.json
