# Round-end check (2 GPUs): GPU suite, smoke, default bench N=1 and N=2, then the profile set of
# the default bench (launch list of the timed step, K1 --set full traffic at b_m 32, attention).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/final_tests.log; tail -3 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench exit $?"
grep '^{' gpurun_out/final_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value'],1), round(d['ms_per_step'],2), d['clocks'], d['roofline']['frac'], d['cpu_baseline'], d['e2e'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/final_bench_n2.log 2>&1; echo "bench n2 exit $?"
grep '^{' gpurun_out/final_bench_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']/d['n_gpus'],1), round(d['ms_per_step'],2))"
B="python bench.py --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv $B --steps 1 --warmup 1 > gpurun_out/ncu_launch_full.log 2>&1; echo "launch list exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tcgen05_pair -s 15 -c 15 -o gpurun_out/k1_full -f $B --layers 1 --mb-per-replica 1 --steps 1 --warmup 1 > gpurun_out/ncu_k1.log 2>&1; echo "k1 full exit $?"
python scripts/ncu_launch_summary.py gpurun_out/launches_full.csv gpurun_out/launch_summary 2 > gpurun_out/launch_summary.log 2>&1; head -14 gpurun_out/launch_summary.log
python scripts/ncu_traffic.py gpurun_out/k1_full.ncu-rep gpurun_out/k1_traffic.json 16384 > gpurun_out/k1_traffic.log 2>&1; tail -1 gpurun_out/k1_traffic.log
