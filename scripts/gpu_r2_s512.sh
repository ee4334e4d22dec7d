#!/bin/bash
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e --no-parity"
for v in main s512; do
  L=""; [ $v != main ] && L="REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so"
  for c in "--config 2 --n-groups 65536" "--config 2 --n-groups 1048576" "--config 3"; do
    env $L timeout 300 $B $c > /tmp/b.json 2>/tmp/b.err
    python -c "import json; d=json.load(open('/tmp/b.json')); print('$v $c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_kernel_ms'].items() if k in ('sweep_hist','sweep_scatter','sweep_accumulate')})" || tail -3 /tmp/b.err
  done
done
