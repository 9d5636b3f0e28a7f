# adjoint knob sweep on config 3 (the r1 sweeps were on config 2) + the new TMA-variant test + ABI
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd_tma.py -m gpu -q --timeout 600 > gpurun_out/y_pytest_tma.log 2>&1; echo "pytest rc=$?" >> gpurun_out/y_pytest_tma.log
PC_FWD_TMA=1 timeout 600 python bench.py --config 3 --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/y_ab_3_tmaenv.log 2>&1
for v in default aw2 aw8 alg4 ach3 ach4 amode1 anolock; do
  E=""; [ $v != default ] && E="PACLOUD_B200_LIB=build/variants/$v.so"
  env $E timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/y_smoke_$v.log
  env $E timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/y_ab_3_$v.log 2>&1
done
echo done
