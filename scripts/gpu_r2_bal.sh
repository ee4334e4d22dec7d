#!/bin/bash
# balanced accumulate schedule (SW_BAL=1, main) vs the 2^19-row item queue (q)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bal
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_parity.py tests/test_gpu_full_size.py tests/test_gpu_split.py -q -p no:cacheprovider -x -k "sweep or partition or config2 or config3 or band or split" > gpurun_out/bal/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bal/pytest.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e --no-parity"
for v in main q; do
  L=""; [ $v != main ] && L="REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so"
  for c in "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576" "--config 3" "--config 2 --n-groups 16384"; do
    env $L timeout 300 $B $c > /tmp/b.json 2>/tmp/b.err
    python -c "import json; d=json.load(open('/tmp/b.json')); print('$v $c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_kernel_ms'].items() if k in ('sweep_hot','sweep_hist','sweep_scatter','sweep_accumulate')})" || tail -3 /tmp/b.err
  done
done
