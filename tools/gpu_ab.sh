# A/B loop: smoke (aborts on failure), GPU tests, config-2 bench per env
# setting, ncu of fwd/adj.  usage: gpu_ab.sh TAG "ENV_A" "ENV_B" ...
TAG=$1; shift
mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1 || { echo "smoke failed rc=$?" >> gpurun_out/smoke_$TAG.log; exit 1; }
i=0
for E in "$@"; do
  env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${TAG}_$i.log 2>&1
  echo "$E" >> gpurun_out/ab_${TAG}_$i.log
  i=$((i+1))
done
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
[ -n "$NCU" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_forward$|k_adjoint" -s 8 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1
echo done
