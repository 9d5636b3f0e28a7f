# round 2: GPU suite, config 5 (clone split) at BASELINE scale, forward variants A/B on config 3
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d_pytest.log
PC_BENCH_DEBUG=1 timeout 1800 python bench.py --config 5 --steps 200 --warmup 3 --no-e2e --no-cpu > gpurun_out/d_bench5_full.log 2>&1; echo "rc=$?" >> gpurun_out/d_bench5_full.log
for v in default w4 c512 c2048 minb2 w4m6; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 600 python bench.py --config 3 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/d_ab_$v.log 2>&1
done
echo done
