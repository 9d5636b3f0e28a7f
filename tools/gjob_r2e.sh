# two-ball adjoint: parity, A/B on configs 3 and 2
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/e_smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py tests/test_gpu_dropins.py -m gpu -q --timeout 900 > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/e_pytest.log
for c in 3 2; do
for v in default old a2m6 a2m8 a2s32 a2s160; do
  E=""; [ $v = old ] && E="PC_ADJ2=0"
  case $v in a2*) E="PACLOUD_B200_LIB=build/variants/$v.so";; esac
  env $E timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/e_ab_${c}_$v.log 2>&1
done
done
echo done
