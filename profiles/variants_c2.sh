# RT0 brick-shape variants (built locally into build_b*/lib.so): bits + bench per variant
mkdir -p gpurun_out/var
python profiles/hash_cfg.py 2 > gpurun_out/var/hash.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-configs > gpurun_out/var/bench_default.log 2>&1
for d in build_b*; do
  HDR_LIB=$d/lib.so python profiles/hash_cfg.py 2 >> gpurun_out/var/hash.txt 2>&1
  HDR_LIB=$d/lib.so timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-configs > gpurun_out/var/bench_$d.log 2>&1
done
