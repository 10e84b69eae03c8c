set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r16.csv $B --layers 4 > gpurun_out/ncu_launch_r16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^gemm_bf16_tcgen05$' -s 8 -c 4 -o gpurun_out/attn_products -f $B --layers 1 > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_rowsoftmax -s 4 -c 2 -o gpurun_out/rowsoftmax2 -f $B --layers 1 > gpurun_out/ncu_rs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tcgen05_pair -s 26 -c 13 -o gpurun_out/pair_te -f $B --layers 1 > gpurun_out/ncu_pair.log 2>&1
ls -la gpurun_out
