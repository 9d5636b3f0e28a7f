# adjoint: 8 balls per warp
mkdir -p gpurun_out
for v in b8w2 b8w4; do
  E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ax_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/ax_smoke_$v.log
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ax_ab_${c}_$v.log 2>&1
  done
done
echo done
