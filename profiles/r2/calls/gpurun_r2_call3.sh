# 1 GPU: K2 forward timing (both shapes) + one ncu --set full capture of attn_fwd2 at the 1.3B shape
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c3_build.log 2>&1
python scripts/attn_bench.py > gpurun_out/c3_attn_bench.jsonl 2>&1
python scripts/attn_bench.py --only 1.3B > gpurun_out/c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_fwd2 -s 1 -c 1 -o gpurun_out/attn_fwd2_r2 \
    python scripts/attn_bench.py --only 1.3B > gpurun_out/c3_ncu.log 2>&1
echo done
