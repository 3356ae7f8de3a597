mkdir -p gpurun_out/r01d
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r01d/bench_cfg$c.log 2>&1
  tail -1 gpurun_out/r01d/bench_cfg$c.log > gpurun_out/r01d/bench_cfg$c.json
done
