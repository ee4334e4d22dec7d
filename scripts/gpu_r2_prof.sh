#!/bin/bash
# Round-2 profiles: ncu --set full of the dominant kernels + config-1 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2p
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e"
python -c "
import paper_1802_09883_b200 as R
print('fp64 adds/s', R.measure_fp_add_rate(R.F64)); print('fp32 adds/s', R.measure_fp_add_rate(R.F32))" > gpurun_out/r2p/fprate.txt 2>&1
cat gpurun_out/r2p/fprate.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p/c1_launches.csv $B --config 1 > /dev/null 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_table -s 3 -c 1 -o gpurun_out/r2p/c1 -f $B --config 1 > gpurun_out/r2p/c1.log 2>&1; echo "c1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_sw_" -s 6 -c 6 -o gpurun_out/r2p/c3 -f $B --config 3 > gpurun_out/r2p/c3.log 2>&1; echo "c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_sw_" -s 6 -c 6 -o gpurun_out/r2p/c2m -f $B --config 2 --n-groups 1048576 > gpurun_out/r2p/c2m.log 2>&1; echo "c2m rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_sw_" -s 6 -c 6 -o gpurun_out/r2p/c2k -f $B --config 2 --n-groups 65536 > gpurun_out/r2p/c2k.log 2>&1; echo "c2k rc=$?"
ls -la gpurun_out/r2p
