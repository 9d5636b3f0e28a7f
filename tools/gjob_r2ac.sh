# ball order: Hilbert (new default) vs Morton, configs 3 / 2 / 4; full GPU suite on the new default
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ac_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ac_smoke.log
for o in hilbert morton; do
  for c in 3 2; do
    PC_BALL_ORDER=$o timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ac_ab_${c}_$o.log 2>&1
  done
  PC_BALL_ORDER=$o timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ac_ab_4_$o.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/ac_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ac_pytest.log
echo done
