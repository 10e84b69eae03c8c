mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c1_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/c1_loopback.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c1_gpu_all.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 scripts/hostlink_probe.py --mb 512 --reps 6 > gpurun_out/hostlink_probe_4gpu_r2.jsonl 2> gpurun_out/hostlink_probe_4gpu_r2.err
echo done
