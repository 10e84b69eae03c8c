mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_attn.py -q -m gpu -s > gpurun_out/attn_tests.log 2>&1; echo "exit $?" >> gpurun_out/attn_tests.log
timeout 120 python scripts/attn_bench.py > gpurun_out/attn_bench.jsonl 2>&1
