# forward setup diet (raw rcp/rsqrt, chunk-local indexing, run range from group spans) + setup unroll
mkdir -p gpurun_out
for v in default nodiet su2 su4; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/z_smoke_$v.log
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/z_ab_${c}_$v.log 2>&1
  done
  env $E timeout 300 python tools/check_fwd_config.py 3 16 > gpurun_out/z_parity_$v.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py tests/test_gpu_fwd_tma.py tests/test_gpu_dropins.py -m gpu -q --timeout 900 > gpurun_out/z_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/z_pytest.log
echo done
