# 1 GPU: K2 tests; forward with the L2-friendly unit order; backward component diagnostics
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c6_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_attn.py -q -x > gpurun_out/c6_attn_tests.log 2>&1
ATTN_EXP_VARIANTS="1 4 8 16 32 64 128 192" ATTN_EXP_B="32" timeout 1200 bash scripts/attn_exp.sh > gpurun_out/c6_attn_exp.jsonl 2> gpurun_out/c6_attn_exp.err
echo done
