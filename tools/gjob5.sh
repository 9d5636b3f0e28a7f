mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/j5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j5_pytest.log
for c in 2 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/j5_bench$c.log 2>&1; done
bash tools/gprof.sh fr2 2 k_fwd_run 8 1
echo done
