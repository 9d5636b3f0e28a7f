# forward defaults XQ + 4 CTAs/SM: full GPU suite, parity, benches, ncu config 3
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/n_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/n_smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/n_pytest.log
for c in 1 2 3 5 4; do timeout 300 python tools/check_fwd_config.py $c 16 >> gpurun_out/n_parity.log 2>&1; done
timeout 900 python bench.py > gpurun_out/n_bench3.log 2>&1
timeout 600 python bench.py --config 2 > gpurun_out/n_bench2.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/n_bench3_ref.log 2>&1
bash tools/gprof.sh n3 3 fwdadj
echo done
