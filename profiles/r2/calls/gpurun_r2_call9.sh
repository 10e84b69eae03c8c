# 4 GPUs: 1-GPU parity subset (GPU 0), the multi-GPU suite, north-star bench lines, host probe at 2 GPUs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c9_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_loopback.py -q > gpurun_out/c9_1gpu.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/c9_multi.log 2>&1
run() { n=$1; port=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n "$@"; }
run 4 29701 > gpurun_out/c9_b12_4x1.jsonl 2> gpurun_out/c9_bench.err
run 4 29702 --offload 1 > gpurun_out/c9_b12_4x1_off.jsonl 2>> gpurun_out/c9_bench.err
run 4 29703 --g-inter 2 > gpurun_out/c9_b12_2x2.jsonl 2>> gpurun_out/c9_bench.err
run 4 29704 --config gpt1.3b > gpurun_out/c9_b13_1x4.jsonl 2>> gpurun_out/c9_bench.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29705 scripts/hostlink_probe.py --mb 512 --reps 6 > gpurun_out/hostlink_probe_2gpu_r2.jsonl 2>> gpurun_out/c9_bench.err
echo done
