#!/bin/bash
cd $GRAFT_REPO_ROOT
N="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e"
KEEP_SOURCE=1 bash scripts/ncu_export.sh c1 -k regex:k_table -s 3 -c 1 $N --config 1
bash scripts/ncu_export.sh g4k -k regex:k_table -s 3 -c 1 $N --config 2 --n-groups 4096
KEEP_SOURCE=1 bash scripts/ncu_export.sh c3hot -k regex:k_sweep_hot -s 3 -c 1 $N --config 3
bash scripts/ncu_export.sh c3 -k regex:"k_sw_hist|k_sweep_cold|k_sweep_acc" -s 3 -c 3 $N --config 3
bash scripts/ncu_export.sh c2m -k regex:"k_sweep_cold|k_sw_hist|k_sweep_acc" -s 3 -c 3 $N --config 2 --n-groups 1048576
bash scripts/ncu_export.sh c2k -k regex:"k_sweep_cold" -s 1 -c 1 $N --config 2 --n-groups 65536
du -sh gpurun_out/prof
