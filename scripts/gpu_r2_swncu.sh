#!/bin/bash
# ncu captures of the sweep path's kernels (config 3 hot pass; G=65536 scatter + accumulate)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sw
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-atomic-baseline --no-configs --no-e2e --no-parity"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep_hot -c 1 -o gpurun_out/sw/hot_c3 $B --config 3 > gpurun_out/sw/n1.log 2>&1; echo "hot rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_cold|k_sweep_acc" -c 2 -o gpurun_out/sw/g65k $B --config 2 --n-groups 65536 > gpurun_out/sw/n2.log 2>&1; echo "g65k rc=$?"
