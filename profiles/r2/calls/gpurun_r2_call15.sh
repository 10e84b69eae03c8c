# 1 GPU: K1 L2 policies + parallel LN-sum final: kernel/step tests, bench x2, K1 traffic capture
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c15_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_loopback.py -q -x > gpurun_out/c15_tests.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c15_bench_a.jsonl 2> gpurun_out/c15_bench.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c15_bench_b.jsonl 2>> gpurun_out/c15_bench.err
B="python bench.py --no-cpu-baseline --e2e-steps 1"
$B --layers 1 --mb-per-replica 1 --steps 1 --warmup 1 > gpurun_out/c15_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:gemm_bf16_tcgen05_pair -s 15 -c 15 -o gpurun_out/k1_full_c15 -f $B --layers 1 --mb-per-replica 1 --steps 1 --warmup 1 > gpurun_out/c15_ncu.log 2>&1
python scripts/ncu_traffic.py gpurun_out/k1_full_c15.ncu-rep gpurun_out/k1_traffic_c15.json 16384 > gpurun_out/c15_traffic.log 2>&1; tail -1 gpurun_out/c15_traffic.log
echo done
