# 2 GPUs: final validation, part 1: build, smoke, the whole -m gpu suite (the 4-GPU cases
# skip here; part 2 runs them), the driver's N = 1 and N = 2 bench commands
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c27_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c27_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c27_gpu_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/c27_bench_n1.jsonl 2> gpurun_out/c27_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/c27_bench_ref_n1.jsonl 2>> gpurun_out/c27_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29841 bench.py --gpus 2 > gpurun_out/c27_bench_n2.jsonl 2>> gpurun_out/c27_bench.err
echo done
