cd $GRAFT_REPO_ROOT
O=gpurun_out/sweep2; mkdir -p $O; : > $O/sweep_c2.jsonl
for G in 1 4 16 64 256 1024 4096 16384 65536 262144 1048576 4194304 16777216; do
  timeout 600 python bench.py --config 2 --n-groups $G --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O/sweep_c2.jsonl 2>> $O/sweep_c2.err
done
wc -l $O/sweep_c2.jsonl
