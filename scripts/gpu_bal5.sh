mkdir -p gpurun_out/tl
b() { name=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 "$@" > gpurun_out/b4_$name.log 2>&1; echo "$name exit $?"
grep '^{' gpurun_out/b4_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$name', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', [round(x,3) for x in d['phases']['bubble_frac_per_rank']])"; }
AXONN_BAL_ATTN_W=1 b gi4_w1 --config gpt12b-pipe --layers 24 --g-inter 4 --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
AXONN_TIMELINE=gpurun_out/tl/gi4_w4 b gi4_w4 --config gpt12b-pipe --layers 24 --g-inter 4 --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
AXONN_BAL_ATTN_W=8 b gi4_w8 --config gpt12b-pipe --layers 24 --g-inter 4 --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
AXONN_TIMELINE=gpurun_out/tl/b24_w4 b 24b_w4 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
AXONN_BAL_ATTN_W=1 b 24b_w1 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline
