# 2 GPUs: final code, whole -m gpu suite (the 4-GPU cases skip) and smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c38_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c38_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c38_gpu_tests.log 2>&1
echo done
