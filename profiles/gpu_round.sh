# round-end evidence on the GPU box: full GPU test suite, smoke, then profiles/collect.sh
R=${1:-r01}
mkdir -p gpurun_out/$R
nvidia-smi > gpurun_out/$R/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$R/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$R/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/$R/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/$R/smoke.log
bash profiles/collect.sh $R > gpurun_out/$R/collect.log 2>&1
bash profiles/stages.sh $R > gpurun_out/$R/stages.log 2>&1
