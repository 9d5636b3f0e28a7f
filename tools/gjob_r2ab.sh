# forward chunk sizes that still fit four CTAs per SM (after the setup diet) + ncu source pass of the new default
mkdir -p gpurun_out
for v in default c1152 c1216 c896; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ab_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/ab_smoke_$v.log
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_ab_${c}_$v.log 2>&1
  done
done
bash tools/gprof.sh ab3 3 fwdadj
echo done
