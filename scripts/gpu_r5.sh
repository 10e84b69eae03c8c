set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for PAIR in 0 1; do for FS in 0 1; do
AXONN_GEMM_PAIR=$PAIR AXONN_FUSED_SOFTMAX=$FS timeout 300 python bench.py --layers 4 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/diag_p${PAIR}_f${FS}.log 2>&1
python -c "
import json,sys
for l in open('gpurun_out/diag_p${PAIR}_f${FS}.log'):
    if l.startswith('{'):
        d=json.loads(l); print('PAIR=$PAIR FS=$FS', round(d['ms_per_step'],1), 'ms', round(d['value'],1), 'TF', 'gemm', round(d['roofline']['achieved'],1))
"
done; done
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k rowsoftmax > gpurun_out/rs.log 2>&1; tail -2 gpurun_out/rs.log
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/gpu_multi.log 2>&1; echo "exit $?" >> gpurun_out/gpu_multi.log
tail -3 gpurun_out/gpu_multi.log
