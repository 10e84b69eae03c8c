mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x > gpurun_out/gpu_k.log 2>&1; echo "exit $?" >> gpurun_out/gpu_k.log
tail -3 gpurun_out/gpu_k.log
for v in 0 4; do DIAG_VARIANT=$v DIAG_ONLY="fc1 fwd" timeout 200 python scripts/diag_sustained.py >> gpurun_out/diag_bn$v.jsonl 2>/dev/null; DIAG_VARIANT=$v DIAG_ONLY="fc2 wgrad" timeout 200 python scripts/diag_sustained.py >> gpurun_out/diag_bn$v.jsonl 2>/dev/null; done
