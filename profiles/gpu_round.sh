mkdir -p gpurun_out/r01b
nvidia-smi > gpurun_out/r01b/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01b/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01b/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r01b/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r01b/smoke.log
bash profiles/collect.sh r01b > gpurun_out/r01b/collect.log 2>&1
