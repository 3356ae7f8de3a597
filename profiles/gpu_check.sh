# quick GPU check: gpu tests + per-config bench lines (no CPU legs) into gpurun_out/$1
set -u
O=gpurun_out/${1:-chk}
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout ${TT:-1200} python -m pytest tests -m gpu -x -q ${PYT:-} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in ${CFGS:-1 2 3 4 5}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu ${BARGS:-} > $O/bench_cfg$c.log 2>&1
done
