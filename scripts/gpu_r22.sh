mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 0 -c 2 -o gpurun_out/attn_bwd -f python scripts/attn_bench.py > gpurun_out/ncu_attn_bwd.log 2>&1
