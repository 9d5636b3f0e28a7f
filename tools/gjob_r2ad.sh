# ball order: Hilbert + radius-sorted runs of 64 / 128 / 256 vs plain Hilbert (configs 3, 2, 4)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ad_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ad_smoke.log
for o in hilbert "hilbert_a0 PC_BALL_SEG=128" "hilbert_a0 PC_BALL_SEG=64" "hilbert_a0 PC_BALL_SEG=256" "hilbert_a0 PC_BALL_SEG=32"; do
  tag=$(echo $o | tr ' =' '__')
  for c in 3 2; do
    env PC_BALL_ORDER=$o timeout 600 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ad_ab_${c}_$tag.log 2>&1
  done
done
for o in hilbert "hilbert_a0 PC_BALL_SEG=128"; do
  tag=$(echo $o | tr ' =' '__')
  env PC_BALL_ORDER=$o timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ad_ab_4_$tag.log 2>&1
done
echo done
