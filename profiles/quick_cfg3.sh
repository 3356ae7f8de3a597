O=gpurun_out/q3; mkdir -p $O
timeout 1800 python -m pytest tests/test_hybridize_gpu.py tests/test_failsafe_gpu.py tests/test_fullsize_gpu.py tests/test_slab.py tests/test_weighted_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -4 $O/pytest.log
for r in 1 2; do timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu --no-configs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['ms_per_step'], d['roofline']['frac'])"; done
