# 1 GPU: the dQ kernel without the acc_done wait too: attention tests, standalone A/B against
# the c19 behaviour (diagnostic build), the 1.3B step
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c39_build.log 2>&1
AXONN_DIAG_DEFINES="-DAXONN_ATTN_NBUF1_WAIT=1" AXONN_DIAG_TAG=_old python -c "from paper_2110_13005_b200 import build as b; b.build(dtypes=('bf16',), force=True)" > gpurun_out/c39_build_old.log 2>&1
timeout 600 python -m pytest tests/test_gpu_attn.py -q > gpurun_out/c39_tests_attn.log 2>&1
for r in 1 2; do
  for sh in 1.3B 12B; do
    timeout 300 python scripts/attn_bench.py --b 32 --only $sh --tag new >> gpurun_out/c39_attn.jsonl 2>> gpurun_out/c39_attn.err
    timeout 300 python scripts/attn_bench.py --b 32 --only $sh --tag old --lib paper_2110_13005_b200/libaxonn_old.so >> gpurun_out/c39_attn.jsonl 2>> gpurun_out/c39_attn.err
  done
done
rm -f paper_2110_13005_b200/libaxonn_old.so
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c39_b13.jsonl 2> gpurun_out/c39_bench.err
echo done
