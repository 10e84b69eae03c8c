# 2 GPUs: L2 policy A/B on one box: none / stream-only / keep+stream, 1.3B N=1 and 12B 2x1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c18_build.log 2>&1
for m in 0 1 2; do
  AXONN_L2_EXP=$m timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c18_b13_l2$m.jsonl 2>> gpurun_out/c18_bench.err
  AXONN_L2_EXP=$m timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29820 + m)) bench.py --gpus 2 > gpurun_out/c18_b12_l2$m.jsonl 2>> gpurun_out/c18_bench.err
done
echo done
