# 2 GPUs: grad_accum_fp32 = 0 (half accumulation, reading D-38): kernel + engine tests, benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c23_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "half_accumulate or remap" > gpurun_out/c23_tests_k.log 2>&1
timeout 900 python -m pytest tests/test_gpu_half_accum.py tests/test_gpu_step.py -q > gpurun_out/c23_tests.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --grad-accum-fp32 0 > gpurun_out/c23_b13_half.jsonl 2> gpurun_out/c23_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 2 --offload 1 --grad-accum-fp32 0 > gpurun_out/c23_b12_2x1_off_half.jsonl 2>> gpurun_out/c23_bench.err
echo done
