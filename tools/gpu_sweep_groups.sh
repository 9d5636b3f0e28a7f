# frame-group overlap sweep on config 2 (bench timing) + engine parity at 4 groups
mkdir -p gpurun_out
for g in ${@:-1 2 4 8}; do
  PC_FRAME_GROUPS=$g timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/groups_$g.log 2>&1
  echo "groups $g rc=$?"
done
PC_FRAME_GROUPS=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "engine" > gpurun_out/groups_test.log 2>&1
