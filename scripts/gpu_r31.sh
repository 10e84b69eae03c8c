mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "stream_k" > gpurun_out/gpu_sk.log 2>&1; echo "exit $?" >> gpurun_out/gpu_sk.log
timeout 600 python -m pytest tests/test_gpu_step.py -q -m gpu -k "overlapped or run_to_run" > gpurun_out/gpu_ov.log 2>&1; echo "exit $?" >> gpurun_out/gpu_ov.log
AXONN_GEMM_SK=0 timeout 600 python -m pytest tests/test_gpu_step.py -q -m gpu -k "overlapped" > gpurun_out/gpu_ov_nosk.log 2>&1; echo "exit $?" >> gpurun_out/gpu_ov_nosk.log
for d in 0 1; do AXONN_GEMM_SK=$d DIAG_ONLY="proj" timeout 120 python scripts/diag_sustained.py >> gpurun_out/diag_sk$d.jsonl 2>/dev/null; AXONN_GEMM_SK=$d DIAG_ONLY="fc1 dgrad" timeout 120 python scripts/diag_sustained.py >> gpurun_out/diag_sk$d.jsonl 2>/dev/null; done
