mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "stream_k or forward or dgrad or wgrad or gelu" > gpurun_out/gpu_sk.log 2>&1; echo "exit $?" >> gpurun_out/gpu_sk.log
tail -3 gpurun_out/gpu_sk.log
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_attn.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python scripts/diag_sustained.py > gpurun_out/diag_sk.jsonl 2>gpurun_out/diag_sk.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1p3b.log 2>&1; echo "exit $?" >> gpurun_out/bench_1p3b.log
