O=gpurun_out/pv2; mkdir -p $O
timeout 1500 python -m pytest tests/test_pencil_gpu.py tests/test_failsafe_gpu.py tests/test_hybridize_gpu.py tests/test_slab.py tests/test_dropin_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for r in 1 2; do
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-configs > $O/base_$r.log 2>&1
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-e2e --no-cpu --no-configs > $O/c1_$r.log 2>&1
done
grep -H -o '"ms_per_step": [0-9.]*' $O/*.log
tail -3 $O/pytest.log
