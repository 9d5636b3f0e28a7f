# refresh: configs 1, 4, 5 (200 iterations), config 3 Gauss N=65, with the current kernels
mkdir -p gpurun_out
timeout 600 python bench.py --config 1 > gpurun_out/r_bench1.log 2>&1
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/r_bench4.log 2>&1
PC_BENCH_DEBUG=1 timeout 1800 python bench.py --config 5 --steps 200 --warmup 3 --no-e2e > gpurun_out/r_bench5.log 2>&1
timeout 1200 python bench.py --config 3 --basis gauss --steps 5 --warmup 3 > gpurun_out/r_bench3g.log 2>&1
echo done
