# usage: tools/gprof.sh TAG CONFIG [fwdadj|all] [basis]
# ncu --set full of the launches inside tools/prof_iter.py's NVTX range;
# exported on the box to gpurun_out/prof_TAG_{raw,src_*}.csv (the .ncu-rep
# itself is kept only when small: gpurun_out travels back capped at 64 MiB)
TAG=$1; C=$2; W=${3:-fwdadj}; BASIS=${4:-polyfourier}
mkdir -p gpurun_out
REP=/tmp/prof_$TAG
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "pc_profile/" -o $REP python tools/prof_iter.py $C $W $BASIS > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
ncu -i $REP.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>>gpurun_out/ncu_$TAG.log
for K in k_fwd_run k_adjoint; do
  ncu -i $REP.ncu-rep --page source --csv -k regex:$K -c 1 > gpurun_out/prof_${TAG}_src_$K.csv 2>>gpurun_out/ncu_$TAG.log
done
SZ=$(stat -c %s $REP.ncu-rep 2>/dev/null || echo 0)
if [ "$SZ" -lt 12000000 ]; then cp $REP.ncu-rep gpurun_out/; fi
ls -la gpurun_out >> gpurun_out/ncu_$TAG.log
