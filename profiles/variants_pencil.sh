# A/B of pencil-kernel builds on config 2 (device-only legs): default lib, then build_b*/libhdr.so
O=gpurun_out/pv; mkdir -p $O
timeout 1500 python -m pytest tests/test_pencil_gpu.py tests/test_failsafe_gpu.py tests/test_hybridize_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for r in 1 2; do
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-configs > $O/base_$r.log 2>&1
for v in build_b[1-5]/; do n=$(basename $v); HDR_LIB=$v/libhdr.so timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-configs > $O/${n}_$r.log 2>&1; done
done
for c in 3 5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-configs > $O/cfg$c.log 2>&1; done
HDR_LIB=build_b6/libhdr.so timeout 300 python bench.py --config 5 --steps 10 --warmup 3 --no-e2e --no-cpu --no-configs > $O/cfg5_nomz.log 2>&1
grep -H -o '"ms_per_step": [0-9.]*' $O/*.log
