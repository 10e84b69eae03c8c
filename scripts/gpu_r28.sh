mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for d in 0 1 3 4; do AXONN_ATTN_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_bwd --csv python scripts/attn_bench.py --only 1.3B 2>/dev/null | grep attn_bwd | awk -F'","' '{print "dbg'$d'", substr($5,1,40), $NF}' >> gpurun_out/attn_dbg.txt; done
