# 2 GPUs: attention backward KA at nv 192 without the acc_done wait (one X / Y buffer): attention
# tests, standalone A/B against the previous behaviour (diagnostic build), the 12B 2x1 step
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c37_build.log 2>&1
AXONN_DIAG_DEFINES="-DAXONN_ATTN_NBUF1_WAIT=1" AXONN_DIAG_TAG=_old python -c "from paper_2110_13005_b200 import build as b; b.build(dtypes=('bf16',), force=True)" > gpurun_out/c37_build_old.log 2>&1
timeout 900 python -m pytest tests/test_gpu_attn.py -q > gpurun_out/c37_tests_attn.log 2>&1
for r in 1 2; do
  for b in 8 32; do
    timeout 300 python scripts/attn_bench.py --b $b --only 12B --tag new >> gpurun_out/c37_attn.jsonl 2>> gpurun_out/c37_attn.err
    timeout 300 python scripts/attn_bench.py --b $b --only 12B --tag old --lib paper_2110_13005_b200/libaxonn_old.so >> gpurun_out/c37_attn.jsonl 2>> gpurun_out/c37_attn.err
  done
done
rm -f paper_2110_13005_b200/libaxonn_old.so
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -k 12b > gpurun_out/c37_tests_full.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 2 > gpurun_out/c37_b12_2x1.jsonl 2> gpurun_out/c37_bench.err
echo done
