# round 2: full GPU suite, NVTX-scoped ncu of configs 2/3 (+ gauss iteration), config 5 at BASELINE scale, gauss config 3 bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_pytest.log
bash tools/gprof.sh c2 2 fwdadj
bash tools/gprof.sh c3 3 fwdadj
bash tools/gprof.sh c3g 3 all gauss
PC_BENCH_DEBUG=1 timeout 1800 python bench.py --config 5 --steps 200 --warmup 3 --no-e2e --no-cpu > gpurun_out/c_bench5_full.log 2>&1; echo "rc=$?" >> gpurun_out/c_bench5_full.log
timeout 1200 python bench.py --config 3 --basis gauss --steps 5 --warmup 3 --no-cpu > gpurun_out/c_bench3_gauss.log 2>&1; echo "rc=$?" >> gpurun_out/c_bench3_gauss.log
echo done
