mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "four_gpus_balanced" > gpurun_out/multi_bal4.log 2>&1; echo "multi exit $?" >> gpurun_out/multi_bal4.log; tail -3 gpurun_out/multi_bal4.log
b() { name=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 "$@" > gpurun_out/b4_$name.log 2>&1; echo "$name exit $?"
grep '^{' gpurun_out/b4_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$name', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', {k: round(v,3) for k,v in d['phases'].items() if isinstance(v,float)})"; }
b 24b_4x1_m64_bal1 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 1
b 24b_4x1_m64_bal0 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 0
b 12b_4x1_off0_bal1 --config gpt12b-pipe --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 1
b 12b_2x2_off0_bal1 --config gpt12b-pipe --g-inter 2 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 1
