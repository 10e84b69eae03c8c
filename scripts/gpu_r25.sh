mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for d in 0 1 2; do AXONN_ATTN_DBG=$d timeout 120 python scripts/attn_bench.py --only 1.3B | sed "s/^/dbg$d /" >> gpurun_out/attn_bench.jsonl 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ --csv python scripts/attn_bench.py --only 1.3B > gpurun_out/attn_launch.csv 2>&1
