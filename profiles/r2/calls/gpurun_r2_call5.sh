# 2 GPUs: multi-GPU suite (fused column reduction vs NCCL, pipelines), then bench lines:
# 1.3B 1x2 fused / nccl, the N=2 default (12B 2x1), the 12B 2x1 with offload
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/c5_multi.log 2>&1
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}"; }
run 29601 --config gpt1.3b > gpurun_out/c5_b13_fused.jsonl 2> gpurun_out/c5_bench.err
AXONN_DP=nccl run 29602 --config gpt1.3b > gpurun_out/c5_b13_nccl.jsonl 2>> gpurun_out/c5_bench.err
run 29603 > gpurun_out/c5_b12_2x1.jsonl 2>> gpurun_out/c5_bench.err
run 29604 --offload 1 > gpurun_out/c5_b12_2x1_off.jsonl 2>> gpurun_out/c5_bench.err
echo done
