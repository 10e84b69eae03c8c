# A/B on one box: bench with the tree's ops.cu (A), then with scripts/ab_ops_old.cu.txt (B), then A again
mkdir -p gpurun_out
bench() { timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$1.log 2>&1; grep '^{' gpurun_out/ab_$1.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"; }
bench A1
cp paper_2110_13005_b200/csrc/ops.cu /tmp/ops_new.cu
cp scripts/ab_ops_old.cu.txt paper_2110_13005_b200/csrc/ops.cu
python -c "from paper_2110_13005_b200 import build; build.build(dtypes=('bf16',))" > /dev/null 2>&1 || echo build-failed
bench B1
cp /tmp/ops_new.cu paper_2110_13005_b200/csrc/ops.cu
python -c "from paper_2110_13005_b200 import build; build.build(dtypes=('bf16',))" > /dev/null 2>&1 || echo build-failed
bench A2
cp scripts/ab_ops_old.cu.txt paper_2110_13005_b200/csrc/ops.cu
python -c "from paper_2110_13005_b200 import build; build.build(dtypes=('bf16',))" > /dev/null 2>&1 || echo build-failed
bench B2
