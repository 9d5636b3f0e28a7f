# adjoint: two neighbouring balls per warp, pair records interleaved per sensor (8 rows per request)
mkdir -p gpurun_out
for v in b2 b2w2; do
  E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/av_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/av_smoke_$v.log
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/av_ab_${c}_$v.log 2>&1
  done
done
PACLOUD_B200_LIB=build/variants/b2.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py tests/test_gpu_dropins.py -m gpu -q --timeout 900 > gpurun_out/av_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/av_pytest.log
echo done
