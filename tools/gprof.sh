# usage: tools/gprof.sh TAG CONFIG KREGEX SKIP COUNT  -> gpurun_out/prof_TAG.ncu-rep
TAG=$1; C=$2; K=$3; S=$4; N=$5
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $N -o gpurun_out/prof_$TAG python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
