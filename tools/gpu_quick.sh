# quick loop: GPU tests + config-2 bench + one ncu capture of fwd/adj
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_forward$|k_adjoint" -s 8 -c 2 -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
