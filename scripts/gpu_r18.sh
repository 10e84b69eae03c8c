set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python scripts/diag_sustained.py > gpurun_out/diag_r18.jsonl 2>gpurun_out/diag_r18.err
for d in 7 8; do for s in "fc1 fwd plain"; do AXONN_GEMM_DBG=$d DIAG_ONLY="$s" timeout 120 python scripts/diag_sustained.py >> gpurun_out/diag_r18_dbg$d.jsonl 2>>gpurun_out/diag_dbg.err; done; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1p3b.log 2>&1; echo "exit $?" >> gpurun_out/bench_1p3b.log
