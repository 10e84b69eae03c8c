set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export AXONN_WATCHDOG_S=300
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/gpu_multi4.log 2>&1; echo "exit $?" >> gpurun_out/gpu_multi4.log
tail -2 gpurun_out/gpu_multi4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4.log 2>&1; echo "exit $?" >> gpurun_out/bench_n4.log
timeout 900 $TR --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.log 2>&1; echo "exit $?" >> gpurun_out/bench_n2.log
timeout 1500 $TR --nproc-per-node 4 --master-port 29605 bench.py --gpus 4 --config gpt12b-pipe --offload 0 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_12b_4x1_off0.log 2>&1; echo "exit $?" >> gpurun_out/bench_12b_4x1_off0.log
timeout 1500 $TR --nproc-per-node 4 --master-port 29606 bench.py --gpus 4 --config gpt12b-pipe --g-inter 2 --offload 0 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_12b_2x2_off0.log 2>&1; echo "exit $?" >> gpurun_out/bench_12b_2x2_off0.log
for f in gpurun_out/bench_n4.log gpurun_out/bench_n2.log gpurun_out/bench_12b_*off0.log; do tail -1 $f | cut -c1-300; done
