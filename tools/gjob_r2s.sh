# final validation: full GPU suite (incl. sharded engine with the 2-collective exchange), launch list of the default bench
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s_smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s_pytest.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s_bench3.log 2>&1; echo "rc=$?" >> gpurun_out/s_bench3.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/s_launches3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/s_ncu_launch3.log 2>&1
echo done
