mkdir -p gpurun_out/q
timeout 900 python -m pytest tests/test_piola_gpu.py tests/test_weighted_gpu.py -x -q -s > gpurun_out/q/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q/pytest.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/q/bench4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spd_hyb|k_piola_gemm" -c 2 -o gpurun_out/q/spd python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/q/ncu.log 2>&1
