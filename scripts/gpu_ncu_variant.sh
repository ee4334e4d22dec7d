# usage: VAR=name bash scripts/gpu_ncu_variant.sh  -> gpurun_out/ncu_$VAR.ncu-rep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export REPRO_B200_LIB=$PWD/scripts/variants/lib_$VAR.so
CMD="python scripts/sweep.py --nobase --variant 1 --groups ${G:-1024}"
$CMD > gpurun_out/plain_$VAR.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:onchip -s 3 -c 1 -o gpurun_out/ncu_$VAR $CMD > gpurun_out/ncu_$VAR.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$VAR.log
