# forced ball-chunk counts on configs 3 and 4 (bench timing, 1 step)
mkdir -p gpurun_out
for c in ${C3:-1 2 4 8}; do
  PC_FWD_CHUNKS=$c timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ch3_$c.log 2>&1
done
for c in ${C4:-1 4 8 16}; do
  PC_FWD_CHUNKS=$c timeout 1200 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ch4_$c.log 2>&1
done
