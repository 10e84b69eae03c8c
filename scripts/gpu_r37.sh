mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_step.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1p3b.log 2>&1; echo "exit $?" >> gpurun_out/bench_1p3b.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ln_|colsum|adamw" --csv python bench.py --layers 2 --mb-per-replica 2 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/small_kernels.csv 2>&1
