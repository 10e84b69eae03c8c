mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for d in 0 7 8; do AXONN_GEMM_DBG=$d timeout 120 python scripts/attn_gemm_diag.py >> gpurun_out/attn_diag.jsonl 2>>gpurun_out/attn_diag.err; done
