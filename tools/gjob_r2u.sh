# forward: per-group full-run ranges (no member test for full groups) - parity + A/B
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/u_smoke.log
for c in 1 2 3 5 4; do timeout 300 python tools/check_fwd_config.py $c 16 >> gpurun_out/u_parity.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -m gpu -q --timeout 900 > gpurun_out/u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/u_pytest.log
for c in 3 2; do
for v in prev default; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/u_ab_${c}_$v.log 2>&1
done
done
echo done
