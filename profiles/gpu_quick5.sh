mkdir -p gpurun_out/q
HDR_LIB=build_x2/libhdr_big.so python profiles/big_timing.py > gpurun_out/q/big_timing.txt 2>&1
timeout 900 python -m pytest tests/test_hybridize_gpu.py tests/test_umma_gpu.py -x -q -s -k "not rt0" > gpurun_out/q/pytest5.log 2>&1; echo "rc=$?" >> gpurun_out/q/pytest5.log
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/q/bench5.log 2>&1
