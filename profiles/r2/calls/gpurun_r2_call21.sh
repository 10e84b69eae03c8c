# 1 GPU: probe 3-D TMA stores (negative / past-extent coordinates), then the remap test under
# compute-sanitizer
mkdir -p gpurun_out
P=scripts/probes/tma3d_store
( for a in "0 0 0" "128 0 0" "-60 1 0" "128 0 0 1" "150 3 32 1" "-60 1 32" "0 4 0"; do timeout 60 $P $a; done ) > gpurun_out/c21_probe.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c21_build.log 2>&1
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_kernels.py -q -x -k "remap_tma and 300" > gpurun_out/c21_sanitizer.log 2>&1
echo done
