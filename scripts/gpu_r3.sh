set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/gpu_multi.log 2>&1; echo "exit $?" >> gpurun_out/gpu_multi.log
tail -3 gpurun_out/gpu_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2.log 2>&1; echo "exit $?" >> gpurun_out/bench_n2.log
tail -2 gpurun_out/bench_n2.log | cut -c1-400
CMD="python bench.py --layers 2 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 800 -c 900 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 40 -c 3 -o gpurun_out/gemm_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 exit $?"
ls -la gpurun_out
