# end-of-session check of the committed state: smoke, full GPU suite, default bench (both arms)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ah_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ah_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/ah_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ah_pytest.log
timeout 900 python bench.py > gpurun_out/ah_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/ah_bench_ref.log 2>&1
echo done
