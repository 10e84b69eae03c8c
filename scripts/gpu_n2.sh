# 2-GPU: fp16 + multi-GPU parity (peer-copy links by default), then 12B 2x1 bench ipc vs nccl
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp16.py -x -q -m gpu > gpurun_out/fp16_tests.log 2>&1; echo "fp16 exit $?" >> gpurun_out/fp16_tests.log; tail -3 gpurun_out/fp16_tests.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "two_gpus or offload" > gpurun_out/multi2.log 2>&1; echo "multi exit $?" >> gpurun_out/multi2.log; tail -5 gpurun_out/multi2.log
for T in ipc nccl; do
AXONN_P2P=$T timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config gpt12b-pipe --g-inter 2 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_12b_2x1_$T.log 2>&1; echo "$T exit $?"
grep '^{' gpurun_out/bench_12b_2x1_$T.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$T', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', d['phases'])"
done
