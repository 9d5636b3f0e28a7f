# config 1 (small) forward chunking sweep
mkdir -p gpurun_out
for c in ${@:-1 2 4 8 16}; do
  PC_FWD_CHUNKS=$c timeout 600 python bench.py --config 1 --steps 2000 --warmup 20 --no-cpu --no-e2e > gpurun_out/c1_$c.log 2>&1
done
