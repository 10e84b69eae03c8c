# 1 GPU: attention tests + timing + trace after the backward handshake changes; loopback + step tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c11_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_attn.py -q -x > gpurun_out/c11_attn_tests.log 2>&1
python scripts/attn_bench.py --b 32 --tag c11 > gpurun_out/c11_attn.jsonl 2>&1
AXONN_DIAG_DEFINES="-DAXONN_ATTN_EXP=256" AXONN_DIAG_TAG=_exp256 python -c "from paper_2110_13005_b200 import build; build.build(dtypes=('bf16',))" > gpurun_out/c11_diag_build.log 2>&1
AXONN_TRACE_FILE=gpurun_out/bwdtrace_c11 python scripts/attn_bench.py --b 32 --only 1.3B --lib paper_2110_13005_b200/libaxonn_exp256.so > gpurun_out/c11_trace.log 2>&1
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_step.py -q > gpurun_out/c11_tests.log 2>&1
echo done
