# 1 GPU: attention tests + timing after the backward unit-order / D-kernel changes; full 1-GPU suite; bench N=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c8_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_attn.py -q -x > gpurun_out/c8_attn_tests.log 2>&1
python scripts/attn_bench.py --b 32 --tag r2c8 > gpurun_out/c8_attn.jsonl 2>&1
python scripts/attn_bench.py --b 8 --tag r2c8 >> gpurun_out/c8_attn.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c8_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/c8_bench.jsonl 2> gpurun_out/c8_bench.err
echo done
