# BASELINE config 2 group-count sweep (2^28 rows, 4^j groups) and config 3,
# one bench.py JSON line each -> gpurun_out/sweep_c2.jsonl, bench_c3.json
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sweep_c2.jsonl
for G in ${GLIST:-1 4 16 64 256 1024 4096 16384 65536 262144 1048576 4194304 16777216}; do
  timeout 600 python bench.py --config 2 --n-groups $G --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline ${PARITY_FLAG} >> gpurun_out/sweep_c2.jsonl 2>> gpurun_out/sweep_c2.err
done
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
