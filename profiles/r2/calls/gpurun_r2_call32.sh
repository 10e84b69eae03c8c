# 1 GPU: K1 operand loads / output stores with a cache_hint only where the policy is not
# evict_normal (A) vs every access hinted (B, -DAXONN_L2_HINT_ALWAYS=1): DRAM bytes of the
# 15 linear-layer GEMMs of a 1-layer 1.3B microbatch (ncu) and the 1.3B step, A B A B
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --e2e-steps 1"
bA() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c32_build_A.log 2>&1; }
bB() { AXONN_DIAG_DEFINES="-DAXONN_L2_HINT_ALWAYS=1" python -c "from paper_2110_13005_b200 import build as b; b.build(force=True)" > gpurun_out/c32_build_B.log 2>&1; }
bA
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k gemm > gpurun_out/c32_tests_k.log 2>&1
for v in A B; do
  b$v
  timeout 900 ncu --set full --clock-control none -k regex:gemm_bf16_tcgen05_pair -s 15 -c 15 -o gpurun_out/c32_k1_$v -f $B --layers 1 --mb-per-replica 1 --steps 1 --warmup 1 > gpurun_out/c32_ncu_$v.log 2>&1
  python scripts/ncu_traffic.py gpurun_out/c32_k1_$v.ncu-rep gpurun_out/c32_k1_traffic_$v.json 16384 > gpurun_out/c32_traffic_$v.log 2>&1; rm -f gpurun_out/c32_k1_$v.ncu-rep
done
for v in A B A B; do
  b$v
  timeout 600 $B >> gpurun_out/c32_bench_$v.jsonl 2>> gpurun_out/c32_bench.err
done
bA
echo done
