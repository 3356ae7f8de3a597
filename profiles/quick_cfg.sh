# one config on the GPU box: its parity tests (pytest -k expression $2) + bench (device-only legs)
C=$1; KEXPR=$2
mkdir -p gpurun_out/c$C
timeout 1200 python -m pytest tests -m gpu -q -x -k "$KEXPR" > gpurun_out/c$C/pytest.log 2>&1; echo rc=$? >> gpurun_out/c$C/pytest.log
for i in 1 2; do
timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu --no-configs > gpurun_out/c$C/bench_$i.log 2>&1
done
