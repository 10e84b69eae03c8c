# 4 GPUs: BASELINE configs[3] proxy (24B layer shape, d 176 -> 192, 6 layers per stage, 4x1,
# b_m 4, offloaded optimizer): microbatch-count sweep m = 16 / 32 / 64 (pipeline bubble), and
# m = 32 with the optimizer in HBM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c33_build.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for m in 16 32 64; do
  timeout 900 $R --master-port $((29890 + m)) bench.py --gpus 4 --config gpt24b-pipe --mb-per-replica $m --steps 3 > gpurun_out/c33_b24_m$m.jsonl 2>> gpurun_out/c33_bench.err
done
timeout 900 $R --master-port 29999 bench.py --gpus 4 --config gpt24b-pipe --offload 0 --steps 3 > gpurun_out/c33_b24_m32_off0.jsonl 2>> gpurun_out/c33_bench.err
echo done
