# G_inter sweep at a fixed model (12B layer shape, 24 layers) and fixed batch (B = 512) on 4 GPUs
mkdir -p gpurun_out
b() { name=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 "$@" > gpurun_out/b4_$name.log 2>&1; echo "$name exit $?"
grep '^{' gpurun_out/b4_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$name', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', {k: (round(v,3) if isinstance(v,float) else v) for k,v in d['phases'].items() if k!='note'})"; }
b sweep_gi1 --config gpt12b-pipe --layers 24 --g-inter 1 --mb-per-replica 16 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
b sweep_gi2 --config gpt12b-pipe --layers 24 --g-inter 2 --mb-per-replica 32 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
b sweep_gi4 --config gpt12b-pipe --layers 24 --g-inter 4 --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
b fp16_12b_2x2 --config gpt12b-pipe --g-inter 2 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --dtype fp16
