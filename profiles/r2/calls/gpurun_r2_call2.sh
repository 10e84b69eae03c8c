# 1 GPU: build, K2 tests first, full GPU suite, bench N=1 default, coarsen-k sweep at 1.3B in HBM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_attn.py -q -x > gpurun_out/c2_attn.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c2_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/c2_bench.jsonl 2> gpurun_out/c2_bench.err
for k in 1 16; do
  timeout 600 python bench.py --coarsen-k $k --no-cpu-baseline > gpurun_out/c2_bench_k$k.jsonl 2>> gpurun_out/c2_bench.err
done
echo done
