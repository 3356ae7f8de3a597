#!/usr/bin/env bash
# Collects the per-round evidence on the GPU box (run from the repo root under
# gpurun):  profiles/collect.sh r01
# Plain runs first; every ncu pass only after its command exited 0 without ncu.
set -u
R=${1:-r01}
OUT=gpurun_out/$R
mkdir -p "$OUT"
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > "$OUT/bench_cfg$c.log" 2>&1
  tail -1 "$OUT/bench_cfg$c.log" > "$OUT/bench_cfg$c.json"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/ref_cfg2.log" 2>&1
tail -1 "$OUT/ref_cfg2.log" > "$OUT/ref_cfg2.json"
timeout 900 python bench.py --impl reference --config 4 --steps 2 --warmup 1 > "$OUT/ref_cfg4.log" 2>&1
tail -1 "$OUT/ref_cfg4.log" > "$OUT/ref_cfg4.json"
# launch list of the headline command (cold, serialised)
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > "$OUT/plain_cfg2.log" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_cfg2.csv" \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > "$OUT/ncu_launch.log" 2>&1
# DRAM traffic of the dominant kernels, one step per config
for c in 2 3 4 5; do
  case $c in
    2) K='regex:k_rt0_pencil|k_rt0_brick|k_rt0_cell|k_rt0_rows' ;;
    3) K='regex:k_hyb_warp' ;;
    4) K='regex:k_piola_gemm|k_spd_hyb|k_run_sum' ;;
    5) K='regex:k_hyb_big|k_gemm_f64' ;;
  esac
  timeout 900 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k "$K" --csv --log-file "$OUT/traffic_cfg$c.csv" \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-configs > "$OUT/ncu_traffic_$c.log" 2>&1
done
# --set full captures of the dominant kernels (summarised by profiles/summarize.py)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rt0_pencil -c 1 \
  -o "$OUT/full_cfg2" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > "$OUT/full2.log" 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_hyb_warp -c 1 \
  -o "$OUT/full_cfg3" python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > "$OUT/full3.log" 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:'^(k_piola_gemm|k_spd_hyb)$' -c 2 \
  -o "$OUT/full_cfg4" python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > "$OUT/full4.log" 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_hyb_big -c 1 \
  -o "$OUT/full_cfg5" python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > "$OUT/full5.log" 2>&1
echo done
