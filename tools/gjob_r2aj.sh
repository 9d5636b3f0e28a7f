# forward: direct threshold 24 as default, dummy-slot queue push variant; parity suite on the default
mkdir -p gpurun_out
for v in default qd; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/aj_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/aj_smoke_$v.log
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/aj_ab_${c}_$v.log 2>&1
  done
  env $E timeout 300 python tools/check_fwd_config.py 3 16 > gpurun_out/aj_parity_$v.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/aj_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/aj_pytest.log
echo done
