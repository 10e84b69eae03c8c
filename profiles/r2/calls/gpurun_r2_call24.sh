# 1 GPU: K1 at the 12B MLP shapes standalone (fc2 dgrad with the DGeLU epilogue vs plain,
# fc1 fwd with GeLU), the half-accumulate kernel test, ncu of the DGeLU dgrad
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c24_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "half_accumulate" > gpurun_out/c24_tests_k.log 2>&1
for sh in "12B fc2 dgrad" "12B fc1 fwd" "12B fc1 dgrad" "12B qkv fwd"; do
  timeout 300 python scripts/microbench.py --what gemm --only "$sh" --variants 0 >> gpurun_out/c24_micro.jsonl 2>> gpurun_out/c24_micro.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tcgen05_pair -c 3 -o gpurun_out/c24_dgelu \
  python scripts/microbench.py --what gemm --only "12B fc2 dgrad" --variants 0 --iters 1 > gpurun_out/c24_ncu.log 2>&1
echo done
