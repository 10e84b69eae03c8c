mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_step.py -x -q -m gpu > gpurun_out/attn_tests.log 2>&1; echo "attn exit $?" >> gpurun_out/attn_tests.log; tail -3 gpurun_out/attn_tests.log
for only in d ka q; do for v in 0 4; do
  echo "== ONLY=$only DBG=$v $(AXONN_ATTN_ONLY=$only AXONN_ATTN_DBG=$v timeout 120 python scripts/attn_bench.py 2>&1 | grep attn_bwd | python -c "import sys,json; print([ (json.loads(l)['shape'], round(json.loads(l)['us'],1)) for l in sys.stdin])")"
done; done
timeout 120 python scripts/attn_bench.py 2>&1
