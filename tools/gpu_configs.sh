mkdir -p gpurun_out
timeout 1200 python bench.py --config 5 --steps 16 --warmup 8 > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
