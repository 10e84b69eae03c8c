# 2 GPUs: half-gradient accumulation over real peer links (2x1 direct send, 1x2 fused reduction)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c36_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "half_accumulation or test_two_gpus" > gpurun_out/c36_tests.log 2>&1
echo done
