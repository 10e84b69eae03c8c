# 2 GPUs: half-accumulation wait moved to the first backward; profile of a middle microbatch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c25_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_half_accum.py -q > gpurun_out/c25_tests.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 2 > gpurun_out/c25_b12_2x1.jsonl 2> gpurun_out/c25_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29832 bench.py --gpus 2 --offload 1 > gpurun_out/c25_b12_2x1_off.jsonl 2>> gpurun_out/c25_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29833 bench.py --gpus 2 --offload 1 --grad-accum-fp32 0 > gpurun_out/c25_b12_2x1_off_half.jsonl 2>> gpurun_out/c25_bench.err
echo done
