mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp16.py -x -q -m gpu > gpurun_out/fp16_tests.log 2>&1; echo "fp16 exit $?" >> gpurun_out/fp16_tests.log; tail -15 gpurun_out/fp16_tests.log
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --dtype fp16 --no-cpu-baseline > gpurun_out/bench_fp16.log 2>&1; echo "bench exit $?"; grep '^{' gpurun_out/bench_fp16.log | head -c 400; tail -3 gpurun_out/bench_fp16.log
