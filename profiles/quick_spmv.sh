O=gpurun_out/spmv; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -k "spmv or pcg or amg or dropin or solve" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -4 $O/pytest.log
for c in 1 2 3 5; do
  timeout 600 python bench.py --config $c --stage spmv --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c spmv', d['ms_per_step'], d['roofline']['frac'], d['config'].get('cuda_graph'))"
  HDR_SPMV_ROWS=1 timeout 600 python bench.py --config $c --stage spmv --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c spmv rows', d['ms_per_step'], d['roofline']['frac'])"
done
