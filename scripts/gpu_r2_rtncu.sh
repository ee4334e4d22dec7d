#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/rtn
RT_N=67108864 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_route -c 1 -o gpurun_out/rtn/route65k python scripts/rt_prof.py 65536 > gpurun_out/rtn/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/rtn/ncu.log
