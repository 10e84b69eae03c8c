set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 300 python bench.py --config tiny --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tiny.log 2>&1; echo "exit $?" >> gpurun_out/bench_tiny.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_1p3b.log 2>&1; echo "exit $?" >> gpurun_out/bench_1p3b.log
tail -3 gpurun_out/smoke.log gpurun_out/bench_tiny.log gpurun_out/bench_1p3b.log
