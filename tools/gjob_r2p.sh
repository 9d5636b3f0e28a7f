# forward/adjoint overlap across frame groups (PC_FRAME_GROUPS) with the current kernels
mkdir -p gpurun_out
for c in 3 2; do
for g in 1 2 4 8; do
  PC_FRAME_GROUPS=$g timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ab_${c}_g$g.log 2>&1
done
done
echo done
