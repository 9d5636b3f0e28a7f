# Full refresh on one B200: tests, smoke, bench (all configs + reference arm),
# ncu launch list and one --set full capture of fwd/adj.  usage: gpu_job.sh TAG
TAG=${1:-run}
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
for c in 1 3 4 5; do
  S=10; [ $c = 1 ] && S=2000; timeout 1500 python bench.py --config $c --steps $S > gpurun_out/bench_c$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c$c.log
done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_forward$|k_adjoint" -s 8 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full.log 2>&1
# every kernel of one config-2 iteration (one launch each) and the config-5
# densify / compaction kernels
timeout 1200 ncu --set full --clock-control none -k regex:"^k_" -s 40 -c 12 -o gpurun_out/prof_${TAG}_all $CMD > gpurun_out/ncu_all.log 2>&1
C5="python bench.py --config 5 --steps 1 --warmup 3 --densify-every 1 --no-e2e --no-cpu"
timeout 600 $C5 > gpurun_out/plain_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:"k_densify|k_scan|k_scatter|k_block|k_gather|k_count|k_prune|k_max" -c 12 -o gpurun_out/prof_${TAG}_c5 $C5 > gpurun_out/ncu_c5.log 2>&1
echo done
