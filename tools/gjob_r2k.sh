# forward: direct-path threshold sweep (DIRECT_MIN 32/28/24/20) - parity + A/B
mkdir -p gpurun_out
for v in dm24; do
  PACLOUD_B200_LIB=build/variants/$v.so timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/k_smoke_$v.log 2>&1
  for c in 1 3; do PACLOUD_B200_LIB=build/variants/$v.so timeout 300 python tools/check_fwd_config.py $c 16 >> gpurun_out/k_parity_$v.log 2>&1; done
done
for c in 3 2; do
for v in default dm28 dm24 dm20; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/k_ab_${c}_$v.log 2>&1
done
done
echo done
