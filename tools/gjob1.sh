mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/j1_smi.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/j1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j1_pytest.log
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu > gpurun_out/j1_bench3.log 2>&1; echo "rc=$?" >> gpurun_out/j1_bench3.log
