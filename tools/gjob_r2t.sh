# capacity buffers: engine/densify tests, sharded, config 5 at BASELINE scale
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_dropins.py tests/test_integration.py -m gpu -q --timeout 900 > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest.log
PC_BENCH_DEBUG=1 timeout 1800 python bench.py --config 5 --steps 200 --warmup 3 --no-e2e > gpurun_out/t_bench5.log 2>&1; echo "rc=$?" >> gpurun_out/t_bench5.log
echo done
