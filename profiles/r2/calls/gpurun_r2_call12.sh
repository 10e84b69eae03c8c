# 2 GPUs: full GPU suite (1-GPU tests on GPU 0 + the 2-GPU tests), bench N=1, bench N=2 default
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c12_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c12_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/c12_bench1.jsonl 2> gpurun_out/c12_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29801 bench.py --gpus 2 > gpurun_out/c12_bench2.jsonl 2>> gpurun_out/c12_bench.err
echo done
