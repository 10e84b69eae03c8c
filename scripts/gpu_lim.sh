mkdir -p gpurun_out
b() { name=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 "$@" > gpurun_out/b4_$name.log 2>&1; echo "$name exit $?"
grep '^{' gpurun_out/b4_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$name', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', {k: round(v,3) for k,v in d['phases'].items() if isinstance(v,float)})"; }
b 24b_lim4 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
b 24b_lim8 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --pipeline-limit 8
b 24b_lim6 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --pipeline-limit 6
