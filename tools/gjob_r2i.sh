# forward: direct full groups (fixed) + combos - parity + A/B
mkdir -p gpurun_out
for v in direct o0c1d o0d; do
  PACLOUD_B200_LIB=build/variants/$v.so timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke_$v.log 2>&1
  for c in 1 3 4; do PACLOUD_B200_LIB=build/variants/$v.so timeout 300 python tools/check_fwd_config.py $c 16 >> gpurun_out/i_parity_$v.log 2>&1; done
done
for c in 3 2; do
for v in default o0c1 direct o0d o0c1d; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/i_ab_${c}_$v.log 2>&1
done
done
echo done
