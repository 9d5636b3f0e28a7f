# forward chunking sweep (target waves of resident CTAs) on configs 2 and 3
mkdir -p gpurun_out
for w in ${@:-1 2 3 4 6}; do
  PC_FWD_WAVES=$w timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/waves_$w.log 2>&1
  PC_FWD_WAVES=$w timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --config 3 > gpurun_out/waves3_$w.log 2>&1
done
