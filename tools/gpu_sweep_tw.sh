# forward segment cap x chunking waves sweep (config 2, bench timing)
mkdir -p gpurun_out
for t in ${TSEGS:-1024}; do for w in ${WAVES:-8 12 16 24}; do
  PC_FWD_TSEG=$t PC_FWD_WAVES=$w timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/tw_${t}_$w.log 2>&1
done; done
