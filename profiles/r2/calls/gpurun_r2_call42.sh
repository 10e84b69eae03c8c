# 4 GPUs: the driver's N = 4 bench on the final code
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c42_build.log 2>&1
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29931 bench.py --gpus 4 > gpurun_out/c42_bench_n4.jsonl 2> gpurun_out/c42_bench.err
echo done
