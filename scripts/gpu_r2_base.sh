#!/bin/bash
# stronger atomicAdd comparators: parity of the baselines + the configs' comparator lines
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -k "atomic" -q -p no:cacheprovider 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-e2e --no-parity"
for c in "--config 3" "--config 2 --n-groups 16" "--config 1" "--config 2 --n-groups 1048576"; do
  timeout 600 $B $c > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c', round(d['ms_per_step'],3), d['baseline_atomic'])" || tail -3 /tmp/b.err
done
