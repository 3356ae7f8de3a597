# A/B of pencil-kernel builds on config 2 (device-only legs): default lib, then build_b*/libhdr.so
O=gpurun_out/pv; mkdir -p $O
for r in 1 2; do
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-configs > $O/base_$r.log 2>&1
for v in build_b*/; do n=$(basename $v); HDR_LIB=$v/libhdr.so timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-configs > $O/${n}_$r.log 2>&1; done
done
grep -h -o '"ms_per_step": [0-9.]*' $O/*.log
