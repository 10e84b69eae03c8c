# 2 GPUs: the driver's N = 2 bench on the final code
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c41_build.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29921 bench.py --gpus 2 > gpurun_out/c41_bench_n2.jsonl 2> gpurun_out/c41_bench.err
echo done
