# Microbatch-size sweep of the 1.3B bench at fixed global batch 64 (G_inter = 1, 1 GPU).
mkdir -p gpurun_out
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/mb_$name.log 2>&1; echo "$name exit $?"
grep '^{' gpurun_out/mb_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$name', round(d['value'],1), 'TF/s', round(d['ms_per_step'],2), 'ms loss', d['loss'], 'mem', round(d['device_mem_gib'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['roofline']['frac'])"; }
b 8 --microbatch 8 --mb-per-replica 8
b 16 --microbatch 16 --mb-per-replica 4
b 32 --microbatch 32 --mb-per-replica 2
b 64 --microbatch 64 --mb-per-replica 1
b 8again --microbatch 8 --mb-per-replica 8
