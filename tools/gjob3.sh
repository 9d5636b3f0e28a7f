mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/j3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j3_pytest.log
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/j3_bench2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_run|k_adjoint" -s 2 -c 2 -o gpurun_out/j3_prof python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/j3_ncu.log 2>&1
echo done
