# final measurements (end of round 2): full GPU suite, default bench (both arms), configs 1/2/4/5, gauss basis,
# launch list + NVTX-scoped ncu of configs 3 and 2
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bb_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/bb_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/bb_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bb_pytest.log
timeout 900 python bench.py > gpurun_out/bb_bench3.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bb_bench3_ref.log 2>&1
timeout 900 python bench.py --config 2 > gpurun_out/bb_bench2.log 2>&1
timeout 900 python bench.py --config 1 > gpurun_out/bb_bench1.log 2>&1
timeout 1500 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bb_bench4.log 2>&1
timeout 1200 python bench.py --config 3 --basis gauss --steps 5 --warmup 3 > gpurun_out/bb_bench3g.log 2>&1
PC_BENCH_DEBUG=1 timeout 1800 python bench.py --config 5 --steps 200 --warmup 3 --no-e2e > gpurun_out/bb_bench5.log 2>gpurun_out/bb_bench5.err; echo "rc=$?" >> gpurun_out/bb_bench5.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/bb_launches3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/bb_ncu_launch3.log 2>&1
bash tools/gprof.sh bb3 3 fwdadj
bash tools/gprof.sh bb2 2 fwdadj
echo done
