#!/bin/bash
# ncu_export.sh NAME NCU-ARGS... -- run ncu --set full into gpurun_out/prof/NAME.ncu-rep,
# export the raw page as CSV and drop the report (gpurun_out/ must stay < 64 MiB)
name=$1; shift
mkdir -p gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -o gpurun_out/prof/$name -f "$@" > gpurun_out/prof/$name.log 2>&1
echo "ncu $name rc=$?"
ncu -i gpurun_out/prof/$name.ncu-rep --page raw --csv > gpurun_out/prof/$name.raw.csv 2>/dev/null
if [ -n "$KEEP_SOURCE" ]; then
  ncu -i gpurun_out/prof/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$name.sass.csv 2>/dev/null
fi
rm -f gpurun_out/prof/$name.ncu-rep
