# forward segment-length sweep on config 2 (bench timing only)
mkdir -p gpurun_out
for t in ${@:-512 768 1024 1280 1536}; do
  PC_FWD_TSEG=$t timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/tseg_$t.log 2>&1
  echo "tseg $t rc=$?"
done
