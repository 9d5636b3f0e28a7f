# adjoint chunk-loop unroll variants - parity smoke + A/B
mkdir -p gpurun_out
for v in au2 au4 ac1u4; do
  PACLOUD_B200_LIB=build/variants/$v.so timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q_smoke_$v.log 2>&1
done
for c in 3 2; do
for v in default au2 au4 ac1u4; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/q_ab_${c}_$v.log 2>&1
done
done
echo done
