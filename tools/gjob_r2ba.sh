# committed tree: smoke + full GPU suite; is the 32-byte sweep start still worth its extra quad now that the L1 pipe is at 74 %?
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ba_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ba_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/ba_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ba_pytest.log
for v in default noal8; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  for c in 3 2; do
    env $E timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ba_ab_${c}_$v.log 2>&1
  done
done
echo done
