# 1-GPU: full-size parity tests, attention-backward variants, optimizer overlap in HBM
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/fullsize.log 2>&1; echo "fullsize exit $?" >> gpurun_out/fullsize.log; tail -3 gpurun_out/fullsize.log
for v in "" "AXONN_ATTN_NFB=2" "AXONN_ATTN_DBG=1" "AXONN_ATTN_DBG=2" "AXONN_ATTN_DBG=4" "AXONN_ATTN_DBG=3"; do
  echo "== $v"; env $v timeout 120 python scripts/attn_bench.py 2>&1 | grep attn_bwd
done > gpurun_out/attn_variants.log 2>&1; cat gpurun_out/attn_variants.log
for ov in 0 1; do
timeout 600 python bench.py --no-cpu-baseline --overlap-next-batch $ov > gpurun_out/bench_ov$ov.log 2>&1; echo "ov$ov exit $?"
grep '^{' gpurun_out/bench_ov$ov.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ov$ov', round(d['value'],1), round(d['ms_per_step'],2), d['phases']['optimizer_exposed_ms'], d['clocks'])"
done
