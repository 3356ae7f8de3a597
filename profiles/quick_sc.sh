O=gpurun_out/sc; mkdir -p $O
timeout 1500 python -m pytest tests/test_condense_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -5 $O/pytest.log
for c in 3; do for s in condense; do
  timeout 600 python bench.py --config $c --stage $s --steps 5 --warmup 2 > $O/stage_cfg${c}_$s.log 2>&1; tail -1 $O/stage_cfg${c}_$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c $s', d['ms_per_step'], d['roofline']['frac'])"
  HDR_SC_NO_WARP=1 timeout 600 python bench.py --config $c --stage $s --steps 5 --warmup 2 > $O/stage_cfg${c}_${s}_old.log 2>&1; tail -1 $O/stage_cfg${c}_${s}_old.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c $s old', d['ms_per_step'], d['roofline']['frac'])"
done; done
