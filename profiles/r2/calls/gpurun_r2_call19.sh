# 2 GPUs: adaptive LN block height: fullsize + step + loopback tests, 12B 2x1 and 1.3B bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c19_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_step.py tests/test_gpu_loopback.py -q > gpurun_out/c19_tests.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 2 > gpurun_out/c19_b12_2x1.jsonl 2> gpurun_out/c19_bench.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c19_b13.jsonl 2>> gpurun_out/c19_bench.err
echo done
