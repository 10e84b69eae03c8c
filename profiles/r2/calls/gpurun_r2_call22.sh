# 2 GPUs: remapped epilogue stored by the epilogue warps from the staging tile
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c22_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/c22_tests_k.log 2>&1 || exit 1
timeout 1500 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_fullsize.py -q > gpurun_out/c22_tests.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 2 > gpurun_out/c22_b12_2x1.jsonl 2> gpurun_out/c22_bench.err
echo done
