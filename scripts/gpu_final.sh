# Round-end check on 2 GPUs: the whole GPU suite (1- and 2-GPU tests), smoke, the default bench line.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/final_tests.log; tail -3 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench exit $?"
grep '^{' gpurun_out/final_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value'],1), round(d['ms_per_step'],2), d['clocks'], d['roofline']['frac'], d['cpu_baseline'], d['e2e'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/final_bench_n2.log 2>&1; echo "bench n2 exit $?"
grep '^{' gpurun_out/final_bench_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']/d['n_gpus'],1), round(d['ms_per_step'],2))"
