mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu -k "not multi and not fullsize" > gpurun_out/gpu1_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu1_tests.log; tail -3 gpurun_out/gpu1_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ln.log 2>&1; echo "bench exit $?"
grep '^{' gpurun_out/bench_ln.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value'],1), round(d['ms_per_step'],2), d['clocks'], {k: v for k, v in d['gemm_breakdown'].items() if 'attn' in k})"
