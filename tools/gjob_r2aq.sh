# adjoint 256-bit loads again on the current code: ptxas's choice (78 registers) and min-blocks 9 (56 registers)
mkdir -p gpurun_out
for v in default v8m9 v8n; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/aq_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/aq_smoke_$v.log
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/aq_ab_${c}_$v.log 2>&1
  done
done
echo done
