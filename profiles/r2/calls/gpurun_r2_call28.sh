# 4 GPUs: final validation, part 2: the multi-GPU parity file on 4 GPUs, the driver's N = 4
# bench, the north-star grid with the offloaded optimizer (fp32 and half accumulation), and the
# G_inter sweep at a fixed batch (Theorem 1 / fig:pipeline-depth at box scale):
# 12B-shaped 16 layers, B = 512 as b_m 8, grids 1x4, 2x2, 4x1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c28_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/c28_gpu_multi.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29851 bench.py --gpus 4 > gpurun_out/c28_bench_n4.jsonl 2> gpurun_out/c28_bench.err
timeout 900 $R --master-port 29852 bench.py --gpus 4 --offload 1 > gpurun_out/c28_b12_4x1_off.jsonl 2>> gpurun_out/c28_bench.err
timeout 900 $R --master-port 29853 bench.py --gpus 4 --offload 1 --grad-accum-fp32 0 > gpurun_out/c28_b12_4x1_off_half.jsonl 2>> gpurun_out/c28_bench.err
for gi in 1 2 4; do
  m=$((64 * gi / 4))
  timeout 900 $R --master-port $((29860 + gi)) bench.py --gpus 4 --config gpt12b --layers 16 --g-inter $gi --mb-per-replica $m --steps 4 > gpurun_out/c28_sweep_gi$gi.jsonl 2>> gpurun_out/c28_bench.err
done
echo done
