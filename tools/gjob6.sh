mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -x > gpurun_out/j6_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j6_pytest.log
for v in default nolpt chunk2k legacy; do
  E=""
  [ $v = nolpt ] && E="PACLOUD_B200_LIB=build/variants/nolpt.so"
  [ $v = chunk2k ] && E="PACLOUD_B200_LIB=build/variants/chunk2k.so"
  [ $v = legacy ] && E="PC_FWD_LEGACY=1"
  for c in 2 3; do env $E timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/j6_${v}_$c.log 2>&1; done
done
timeout 900 python -m pytest tests/test_gpu_sharded.py -q --timeout 900 > gpurun_out/j6_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/j6_sharded.log
echo done
