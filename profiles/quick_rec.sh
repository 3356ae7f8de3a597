O=gpurun_out/rec; mkdir -p $O
timeout 1500 python -m pytest tests/test_hybridize_gpu.py tests/test_fullsize_gpu.py tests/test_failsafe_gpu.py tests/test_dropin_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -4 $O/pytest.log
for c in 3 1; do timeout 600 python bench.py --config $c --stage recover --steps 5 --warmup 2 > $O/stage_cfg${c}_recover.log 2>&1; tail -1 $O/stage_cfg${c}_recover.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c recover', d['ms_per_step'], d['roofline']['frac'])"; done
