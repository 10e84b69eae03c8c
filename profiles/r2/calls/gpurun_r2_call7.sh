# 1 GPU: ncu --set full of the attention backward kernels (KA and !KA) at the 1.3B shape, b = 8
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c7_build.log 2>&1
python scripts/attn_bench.py --only 1.3B > gpurun_out/c7_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 3 -c 3 -o gpurun_out/attn_bwd_r2 \
    python scripts/attn_bench.py --only 1.3B > gpurun_out/c7_ncu.log 2>&1
echo done
