# forward variants: MUFU seeds from the setup, chunk 512, TMA-staged ball tiles
mkdir -p gpurun_out
for v in default seeds c512 c512s tma512 tma512s tma1024; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/w_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/w_smoke_$v.log
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/w_ab_${c}_$v.log 2>&1
  done
  env $E timeout 300 python tools/check_fwd_config.py 3 16 > gpurun_out/w_parity_$v.log 2>&1
done
echo done
