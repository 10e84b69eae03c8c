mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_attn.py tests/test_gpu_step.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_1p3b.log 2>&1; echo "exit $?" >> gpurun_out/bench_1p3b.log
