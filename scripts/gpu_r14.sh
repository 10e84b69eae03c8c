set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python scripts/diag_sustained.py > gpurun_out/diag_sustained.jsonl 2> gpurun_out/diag_sustained.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1p3b.log 2>&1; echo "exit $?" >> gpurun_out/bench_1p3b.log
