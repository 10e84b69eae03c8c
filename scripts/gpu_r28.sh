mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_attn.py tests/test_gpu_step.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1p3b.log 2>&1; echo "exit $?" >> gpurun_out/bench_1p3b.log
for d in 0 1 3 4; do AXONN_ATTN_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_bwd --csv python scripts/attn_bench.py --only 1.3B 2>/dev/null | grep attn_bwd | awk -F'","' '{print "dbg'$d'", substr($5,1,40), $NF}' >> gpurun_out/attn_dbg.txt; done
