# Round-2 profile set of the default bench (1 GPU): launch list of the timed step (ncu, serialised,
# compare shares), K1 --set full traffic of one 1-layer b_m 32 microbatch, K2 forward --set full.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/prof_build.log 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 1"
$B --steps 1 --warmup 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv $B --steps 1 --warmup 1 > gpurun_out/ncu_launch_r2.log 2>&1; echo "launch list exit $?"
$B --layers 1 --mb-per-replica 1 --steps 1 --warmup 1 > gpurun_out/prof_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tcgen05_pair -s 15 -c 15 -o gpurun_out/k1_full_r2 -f $B --layers 1 --mb-per-replica 1 --steps 1 --warmup 1 > gpurun_out/ncu_k1_r2.log 2>&1; echo "k1 full exit $?"
python scripts/ncu_launch_summary.py gpurun_out/launches_r2.csv gpurun_out/launch_summary_r2 2 > gpurun_out/launch_summary_r2.log 2>&1; head -20 gpurun_out/launch_summary_r2.log
python scripts/ncu_traffic.py gpurun_out/k1_full_r2.ncu-rep gpurun_out/k1_traffic_r2.json 16384 > gpurun_out/k1_traffic_r2.log 2>&1; tail -1 gpurun_out/k1_traffic_r2.log
python scripts/attn_bench.py --b 32 --only 1.3B > gpurun_out/prof_plain3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd2 -s 1 -c 1 -o gpurun_out/attn_fwd2_b32_r2 -f python scripts/attn_bench.py --b 32 --only 1.3B > gpurun_out/ncu_attn_r2.log 2>&1; echo "attn exit $?"
echo done
