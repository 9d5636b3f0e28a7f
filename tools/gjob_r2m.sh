# forward: quarter transposes (9 KB) and 4 CTAs/SM; run vs pool kernels
mkdir -p gpurun_out
for v in xq xq4; do
  PACLOUD_B200_LIB=build/variants/$v.so timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke_$v.log 2>&1
  for c in 1 3; do PACLOUD_B200_LIB=build/variants/$v.so PC_FWD_POOL=0 timeout 300 python tools/check_fwd_config.py $c 16 >> gpurun_out/m_parity_$v.log 2>&1; done
done
for c in 3 2; do
for v in default xq xq4; do
 for P in 0 1; do
  E="PC_FWD_POOL=$P"; [ $v != default ] && E="$E PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/m_ab_${c}_${v}_p$P.log 2>&1
 done
done
done
echo done
