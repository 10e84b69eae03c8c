# 1 GPU: step / loopback / full-size parity on the final attention backward
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c40_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_loopback.py tests/test_gpu_fullsize.py tests/test_gpu_half_accum.py tests/test_gpu_fp16.py -q > gpurun_out/c40_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c40_smoke.log 2>&1
echo done
