# 1 GPU: loopback bitwise diagnosis; backward timeline trace (diagnostic build); attention tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c10_build.log 2>&1
timeout 600 python scripts/debug_loopback_bitwise.py 4 > gpurun_out/c10_debug_loop.log 2>&1
timeout 600 python scripts/debug_loopback_bitwise.py 2 >> gpurun_out/c10_debug_loop.log 2>&1
AXONN_DIAG_DEFINES="-DAXONN_ATTN_EXP=256" AXONN_DIAG_TAG=_exp256 python -c "from paper_2110_13005_b200 import build; build.build(dtypes=('bf16',))" > gpurun_out/c10_diag_build.log 2>&1
AXONN_TRACE_FILE=gpurun_out/bwdtrace_b32 python scripts/attn_bench.py --b 32 --only 1.3B --lib paper_2110_13005_b200/libaxonn_exp256.so > gpurun_out/c10_trace.log 2>&1
timeout 600 python -m pytest tests/test_gpu_loopback.py -q -k direct > gpurun_out/c10_direct.log 2>&1
echo done
