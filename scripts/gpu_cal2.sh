# Speed-weighted split on a clean 4-GPU box: the calibrated-split tests, then 24B 4x1 balanced
# (FLOP model) vs calibrated.  nvidia-smi first: no other process on the GPUs.
mkdir -p gpurun_out
nvidia-smi --query-compute-apps=pid,used_memory --format=csv > gpurun_out/cal2_apps_before.txt
timeout 600 python -m pytest -q -m gpu tests/test_gpu_multi.py -k "speed_weighted or calibrated" tests/test_gpu_kernels.py -k "calibrate or speed" > gpurun_out/cal2_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/cal2_tests.log
nvidia-smi --query-compute-apps=pid,used_memory --format=csv > gpurun_out/cal2_apps_after.txt; cat gpurun_out/cal2_apps_after.txt
b() { name=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 "$@" > gpurun_out/cal2_$name.log 2>&1; echo "$name exit $?"
grep '^{' gpurun_out/cal2_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); c=d['config']; print('$name', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', [round(x,3) for x in d['phases']['bubble_frac_per_rank']], c['stage_blocks'], c['stage_speed_tflops'])"; }
b 24b_bal1 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 1
b 24b_bal2 --config gpt24b-pipe --mb-per-replica 64 --offload 0 --steps 2 --warmup 3 --no-cpu-baseline --stage-balance 2
