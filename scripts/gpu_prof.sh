# Round-end profile set (1 GPU): launch list of the bench command, ncu --set full of one
# microbatch's K1 launches (roofline traffic) and of the fused attention kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
B="python bench.py --no-cpu-baseline --e2e-steps 1"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv $B --steps 1 --warmup 1 > gpurun_out/ncu_launch_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tcgen05_pair -s 15 -c 15 -o gpurun_out/k1_full -f $B --layers 1 --mb-per-replica 1 --steps 1 --warmup 1 > gpurun_out/ncu_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 5 -c 5 -o gpurun_out/attn_full -f $B --layers 1 --mb-per-replica 1 --steps 1 --warmup 1 > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
python scripts/ncu_launch_summary.py gpurun_out/launches_full.csv gpurun_out/launch_summary 8 > gpurun_out/launch_summary.log 2>&1; head -30 gpurun_out/launch_summary.log
python scripts/ncu_traffic.py gpurun_out/k1_full.ncu-rep gpurun_out/k1_traffic.json > gpurun_out/k1_traffic.log 2>&1; tail -3 gpurun_out/k1_traffic.log
