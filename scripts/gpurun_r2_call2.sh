# 1 GPU: build, full GPU suite, bench N=1 default, coarsen-k sweep at 1.3B in HBM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/c2_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/c2_bench.jsonl 2> gpurun_out/c2_bench.err
for k in 1 16; do
  timeout 600 python bench.py --coarsen-k $k --no-cpu-baseline > gpurun_out/c2_bench_k$k.jsonl 2>> gpurun_out/c2_bench.err
done
echo done
