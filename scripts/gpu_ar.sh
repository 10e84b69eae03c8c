# 2-GPU: overlapped column all-reduce (parity + bitwise) and the 1.3B DP bench variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "bitwise or 1-2" > gpurun_out/multi_ar.log 2>&1; echo "multi exit $?" >> gpurun_out/multi_ar.log; tail -5 gpurun_out/multi_ar.log
run() { env $1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/bench_n2_$2.log 2>&1; echo "$2 exit $?"
grep '^{' gpurun_out/bench_n2_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$2', round(d['value']/d['n_gpus'],1), 'TF/s/GPU', round(d['ms_per_step'],1), 'ms', 'ar_exposed', round(d['phases']['allreduce_exposed_ms'],2), 'opt', round(d['phases']['optimizer_exposed_ms'],2), 'e2e', round(d['e2e']['value']/d['n_gpus'],1))"; }
run AXONN_AR_OVERLAP=0 ov0
run AXONN_AR_OVERLAP=1 ov1
run "AXONN_AR_OVERLAP=1 AXONN_DP_CTAS=8" ov1c8
run "AXONN_AR_OVERLAP=1 AXONN_DP_CTAS=16" ov1c16
