# round-2 status check: smoke, GPU tests, bench configs 2/3 (register-run forward vs legacy)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/a_smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
for c in 2 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/a_bench$c.log 2>&1
  PC_FWD_LEGACY=1 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/a_bench${c}_legacy.log 2>&1
done
for c in 1 2 3 5 4; do
  timeout 300 python tools/check_fwd_config.py $c 16 >> gpurun_out/a_parity.log 2>&1
done
echo done
