# 2 GPUs: multi-GPU parity on the final code (2-GPU cases of the multi file)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c43_build.log 2>&1
timeout 420 python -m pytest tests/test_gpu_multi.py -q -x -k "test_two_gpus or half_accumulation or fused_column" > gpurun_out/c43_tests.log 2>&1
echo done
