#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof8
for v in head tb0; do
  if [ $v = head ]; then cmd="python scripts/variants/headpkg/sweep_head.py --nobase --groups 1024"; lib=""; else cmd="python scripts/sweep.py --nobase --groups 1024"; lib="REPRO_B200_LIB=$PWD/scripts/variants/lib_$v.so"; fi
  env $lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_table -s 3 -c 1 -o gpurun_out/prof8/$v -f $cmd > gpurun_out/prof8/$v.log 2>&1; echo "$v rc=$?"
  ncu -i gpurun_out/prof8/$v.ncu-rep --page raw --csv > gpurun_out/prof8/$v.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof8/$v.ncu-rep --page source --csv --print-source sass > gpurun_out/prof8/$v.sass.csv 2>/dev/null
  rm -f gpurun_out/prof8/$v.ncu-rep
done
