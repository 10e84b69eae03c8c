# 1 GPU: output eviction policy only for > 100 MB outputs: bench x2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c16_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/c16_tests.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c16_bench_a.jsonl 2> gpurun_out/c16_bench.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c16_bench_b.jsonl 2>> gpurun_out/c16_bench.err
echo done
