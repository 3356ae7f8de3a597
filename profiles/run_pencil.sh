# pencil kernel round trip on the GPU box: RT0 parity tests, bench lines, launch list, traffic, one full capture
O=gpurun_out/p4; mkdir -p $O
timeout 1200 python -m pytest tests/test_pencil_gpu.py tests/test_failsafe_gpu.py tests/test_hybridize_gpu.py tests/test_condense_gpu.py tests/test_dropin_gpu.py tests/test_slab.py tests/test_fullsize_gpu.py -m gpu -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for c in 2 1; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 > $O/bench_c$c.log 2>&1; tail -1 $O/bench_c$c.log > $O/bench_cfg$c.json; done
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
timeout 900 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:k_rt0 --csv --log-file $O/traffic_cfg2.csv python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu --no-configs > $O/ncu_traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rt0_pencil -c 1 \
  -o $O/full_cfg2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > $O/full2.log 2>&1
ncu -i $O/full_cfg2.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/full_cfg2.ncu-rep --page source --csv > $O/source.csv 2>/dev/null
echo done
