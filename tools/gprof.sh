# usage: tools/gprof.sh TAG CONFIG [fwdadj|all] -> gpurun_out/prof_TAG.ncu-rep
# (ncu --set full of the launches inside tools/prof_iter.py's NVTX range)
TAG=$1; C=$2; W=${3:-fwdadj}; BASIS=${4:-polyfourier}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "pc_profile/" -o gpurun_out/prof_$TAG python tools/prof_iter.py $C $W $BASIS > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
