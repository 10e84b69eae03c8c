# 1 GPU: build; K2 + loopback (incl. fused column reduction) + step tests; K2 diagnostic variants
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c4_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_loopback.py tests/test_gpu_step.py -q -x > gpurun_out/c4_tests.log 2>&1
timeout 900 bash scripts/attn_exp.sh > gpurun_out/c4_attn_exp.jsonl 2> gpurun_out/c4_attn_exp.err
echo done
