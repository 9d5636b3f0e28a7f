# Functional check of the N>1 bench path on one GPU (gloo, 2 ranks sharing
# cuda:0): frame sharding (configs 2, 5), sensor sharding (configs 1, 4) and
# the reference arm.  Not a measurement.
mkdir -p gpurun_out
run() {  # name port args...
  local name=$1 port=$2; shift 2
  PC_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 "$@" > gpurun_out/mr_$name.log 2>&1
  echo "$name rc=$?" >> gpurun_out/mr_$name.log
}
run c2 29611 --steps 2 --warmup 3 --no-cpu
run c1 29612 --steps 2 --warmup 3 --no-cpu --config 1
run c5 29613 --steps 2 --warmup 3 --no-cpu --no-e2e --config 5 --densify-every 2
run c4 29614 --steps 1 --warmup 3 --no-cpu --no-e2e --config 4
run ref 29615 --impl reference --steps 1 --warmup 1
