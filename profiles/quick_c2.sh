# config-2 check on the GPU box: k = 0 parity tests + bench (device-only legs); $1 = extra lib variant dir
mkdir -p gpurun_out/c2
timeout 900 python -m pytest tests/test_hybridize_gpu.py tests/test_fullsize_gpu.py tests/test_failsafe_gpu.py -q -x -k "rt0 or k0 or 0-64 or cfg1 or cfg2 or golden or reference or pattern or values" > gpurun_out/c2/pytest.log 2>&1; echo rc=$? >> gpurun_out/c2/pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-configs > gpurun_out/c2/bench_$i.log 2>&1
for v in "$@"; do HDR_LIB=$v/lib.so timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-configs > gpurun_out/c2/bench_$(basename $v)_$i.log 2>&1; done
done
