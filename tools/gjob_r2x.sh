# forward: chunk size at 3 CTAs / SM, L1 prefetch, TMA at chunk 768; ncu source pass of the default build
mkdir -p gpurun_out
for v in default c2048m3 c1536m3 c1024m3 pf tma768m3; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/x_smoke_$v.log
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/x_ab_${c}_$v.log 2>&1
  done
done
bash tools/gprof.sh x3 3 fwdadj
echo done
