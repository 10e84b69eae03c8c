set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max --format=csv > gpurun_out/probe_smi.csv 2>&1
nproc > gpurun_out/probe_nproc.txt; free -g >> gpurun_out/probe_nproc.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/r1_kernels.log 2>&1
echo "exit $?" >> gpurun_out/r1_kernels.log
tail -30 gpurun_out/r1_kernels.log
