O=gpurun_out/sc; mkdir -p $O
timeout 1500 python -m pytest tests/test_condense_gpu.py tests/test_fullsize_gpu.py tests/test_dropin_gpu.py tests/test_essential_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -15 $O/pytest.log
for c in 2 1 3; do for s in condense; do
  timeout 600 python bench.py --config $c --stage $s --steps 5 --warmup 2 > $O/stage_cfg${c}_$s.log 2>&1; tail -1 $O/stage_cfg${c}_$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c $s', d['ms_per_step'], d['roofline']['frac'])"
done; done
HDR_SC_NO_PENCIL=1 timeout 600 python bench.py --config 2 --stage condense --steps 5 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 condense old', d['ms_per_step'], d['roofline']['frac'])"
