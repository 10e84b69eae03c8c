set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
export AXONN_WATCHDOG_S=300
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/gpu_multi4.log 2>&1; echo "exit $?" >> gpurun_out/gpu_multi4.log
tail -2 gpurun_out/gpu_multi4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n4.log 2>&1; echo "exit $?" >> gpurun_out/bench_n4.log
timeout 1500 $TR --nproc-per-node 4 --master-port 29605 bench.py --gpus 4 --config gpt12b-pipe --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_12b_4x1_off1.log 2>&1; echo "exit $?" >> gpurun_out/bench_12b_4x1_off1.log
timeout 1500 $TR --nproc-per-node 4 --master-port 29606 bench.py --gpus 4 --config gpt12b-pipe --g-inter 2 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_12b_2x2_off1.log 2>&1; echo "exit $?" >> gpurun_out/bench_12b_2x2_off1.log
timeout 1500 $TR --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 --config gpt24b-pipe --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_24b_4x1_off1.log 2>&1; echo "exit $?" >> gpurun_out/bench_24b_4x1_off1.log
for f in gpurun_out/bench_n4.log gpurun_out/bench_12b_*.log gpurun_out/bench_24b_*.log; do tail -1 $f | cut -c1-300; done
