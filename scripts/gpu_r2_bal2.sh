#!/bin/bash
# accumulate schedule variants (main: cost-balanced cuts, publish = 2^17 rows; pb0: row-balanced; pb18: 2^18;
# q: 2^19-row item queue) and warp-match scatter ranks (mr); sparse path with the own radix sort
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bal2
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_band.py tests/test_gpu_full_size.py -q -p no:cacheprovider -x > gpurun_out/bal2/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bal2/pytest.txt
REPRO_B200_LIB=$PWD/scripts/variants/lib_mr.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_band.py -q -p no:cacheprovider -x -k "sweep or partition or band" > gpurun_out/bal2/pytest_mr.txt 2>&1; echo "pytest mr rc=$?"; tail -2 gpurun_out/bal2/pytest_mr.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e --no-parity"
for v in main pb0 pb18 q mr; do
  L=""; [ $v != main ] && L="REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so"
  for c in "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576" "--config 3" "--config 2 --n-groups 16384" "--config 2 --n-groups 262144"; do
    env $L timeout 300 $B $c > /tmp/b.json 2>/tmp/b.err
    python -c "import json; d=json.load(open('/tmp/b.json')); print('$v $c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_kernel_ms'].items() if k in ('sweep_hot','sweep_hist','sweep_scatter','sweep_accumulate')})" || tail -3 /tmp/b.err
  done
done
timeout 600 python -c "import json, torch, bench, paper_1802_09883_b200 as R; d=bench.run_sparse(R, torch, 5, 3); print('f1', d['ms_per_step'], d.get('parity'))"; echo "f1 rc=$?"
