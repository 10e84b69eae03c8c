# 2 GPUs: 1.3B microbatch choice on the current build (b_m 32 x 2 vs 64 x 1 vs 16 x 4) and the N = 2 default
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c17_build.log 2>&1
for mb in 64 16 32; do
  timeout 600 python bench.py --no-cpu-baseline --microbatch $mb --mb-per-replica $((64 / mb)) > gpurun_out/c17_b13_mb$mb.jsonl 2>> gpurun_out/c17_bench.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 > gpurun_out/c17_b12_2x1.jsonl 2>> gpurun_out/c17_bench.err
echo done
