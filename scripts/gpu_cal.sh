# Round 56: speed-weighted stage split (reading D-21c) on 4 GPUs + new tests + the new default bench.
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_kernels.py -k calibrate tests/test_gpu_multi.py -k "speed_weighted or calibrated or balanced" > gpurun_out/cal_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/cal_tests.log
b() { name=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 "$@" > gpurun_out/cal_$name.log 2>&1; echo "$name exit $?"
grep '^{' gpurun_out/cal_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); c=d['config']; print('$name', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', [round(x,3) for x in d['phases']['bubble_frac_per_rank']], c['stage_blocks'], c['stage_speed_tflops'])"; }
b 24b_bal1 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 1
b 24b_bal2 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 2
b 12b_bal1 --config gpt12b-pipe --layers 24 --g-inter 4 --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 1
b 12b_bal2 --config gpt12b-pipe --layers 24 --g-inter 4 --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 2
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_fullsize.py > gpurun_out/cal_fullsize.log 2>&1; echo "fullsize exit $?"; tail -2 gpurun_out/cal_fullsize.log
