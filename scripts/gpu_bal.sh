mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "balanced or two_gpus" > gpurun_out/multi_bal.log 2>&1; echo "multi exit $?" >> gpurun_out/multi_bal.log; tail -4 gpurun_out/multi_bal.log
timeout 300 python -m pytest tests/test_gpu_step.py -x -q -m gpu > gpurun_out/step.log 2>&1; echo "step exit $?"; tail -1 gpurun_out/step.log
for B in 1 0; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config gpt12b-pipe --g-inter 2 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance $B > gpurun_out/bench_12b_2x1_bal$B.log 2>&1; echo "bal$B exit $?"
grep '^{' gpurun_out/bench_12b_2x1_bal$B.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bal$B', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', {k: round(v,3) for k,v in d['phases'].items() if isinstance(v,float)})"
done
