mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 0 -c 6 -o gpurun_out/attn_all -f python scripts/attn_bench.py --only 1.3B > gpurun_out/ncu_attn_all.log 2>&1
