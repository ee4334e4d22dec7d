#!/bin/bash
# ncu --set full of the dominant kernels of the remaining bench sub-results at HEAD (DRAM traffic per launch for
# roofline.traffic): config 3 hot pass, config 4 k_lean_multi, config 2 at G = 16 (lean), 4096 (k_table band), 2^20 (scatter)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu5; mkdir -p $O
Q="--steps 1 --warmup 3 --no-cpu-baseline --no-parity --no-atomic-baseline --no-configs --no-e2e"
N="ncu --set full --clock-control none -f"
timeout 600 $N -k regex:k_sweep_hot -s 3 -c 1 -o $O/c3_hot python bench.py --config 3 $Q > $O/c3.log 2>&1; echo "c3 rc=$?"
timeout 900 $N -k regex:k_lean_multi -s 3 -c 1 -o $O/c4_lean python bench.py --config 4 $Q > $O/c4.log 2>&1; echo "c4 rc=$?"
timeout 600 $N -k regex:k_lean_multi -s 3 -c 1 -o $O/g16_lean python bench.py --config 2 --n-groups 16 $Q > $O/g16.log 2>&1; echo "g16 rc=$?"
timeout 600 $N -k regex:k_table -s 3 -c 1 -o $O/g4096_table python bench.py --config 2 --n-groups 4096 $Q > $O/g4096.log 2>&1; echo "g4096 rc=$?"
timeout 600 $N -k regex:k_table -s 3 -c 1 -o $O/g1024_table python bench.py --config 2 --n-groups 1024 $Q > $O/g1024.log 2>&1; echo "g1024 rc=$?"
timeout 600 $N -k regex:"k_sweep_cold|k_sweep_acc" -c 2 -o $O/g1m_sweep python bench.py --config 2 --n-groups 1048576 $Q > $O/g1m.log 2>&1; echo "g1m rc=$?"
for r in $O/*.ncu-rep; do python scripts/ncu_summary.py $r > ${r%.ncu-rep}.txt 2>&1; rm -f $r; done
ls -la $O
