# Build a variant of libpacloud_b200.so with extra nvcc defines into
# build/variants/NAME.so (select it with PACLOUD_B200_LIB=...).
# usage: tools/build_variant.sh NAME "-DPC_X=1 -DPC_Y=2"
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2412_03898_b200/csrc
OUT=$ROOT/build/variants/$NAME
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$ROOT/include $DEFS"
for f in radiator fwd_run deform optim voxel ubp; do
  nvcc $FL -c $C/$f.cu -o $OUT/$f.o &
done
nvcc $FL -DPC_FR_NS=tma -DPC_FR_TMA=1 -DPC_FR_CHUNK=512 -c $C/fwd_run.cu -o $OUT/fwd_run_tma.o &
wait
nvcc $ARCH -shared -cudart static -o $ROOT/build/variants/$NAME.so $OUT/*.o
echo built build/variants/$NAME.so
