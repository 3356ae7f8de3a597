# A/B of k_sc_warp builds on config 3 condensation: default lib, then build_b*/libhdr.so
O=gpurun_out/scv; mkdir -p $O
for r in 1 2; do
timeout 300 python bench.py --config 3 --stage condense --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('base', d['ms_per_step'])"
for v in build_b*/; do n=$(basename $v); HDR_LIB=$v/libhdr.so timeout 300 python bench.py --config 3 --stage condense --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['ms_per_step'])"; done
done
