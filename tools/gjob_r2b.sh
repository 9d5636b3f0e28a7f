# round 2: new parity tests, config-3 headline bench + reference arm, ncu (launch list + full) on configs 2/3
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dropins.py tests/test_integration.py tests/test_gpu_fullsize.py -m gpu -q --timeout 900 -rs > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b_pytest.log
timeout 900 python bench.py > gpurun_out/b_bench3.log 2>&1; echo "rc=$?" >> gpurun_out/b_bench3.log
timeout 900 python bench.py --impl reference > gpurun_out/b_bench3_ref.log 2>&1; echo "rc=$?" >> gpurun_out/b_bench3_ref.log
timeout 600 python bench.py --config 2 > gpurun_out/b_bench2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/b_launches3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/b_ncu_launch3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/b_launches2.csv python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/b_ncu_launch2.log 2>&1
bash tools/gprof.sh c2 2 "k_fwd_run|k_adjoint" 2 2
bash tools/gprof.sh c3 3 "k_fwd_run|k_adjoint" 2 2
nproc > gpurun_out/b_nproc.txt
timeout 1200 python tools/ref_full.py 2 3 > gpurun_out/b_ref_full2.log 2>&1
echo done
