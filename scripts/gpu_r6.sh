set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export AXONN_WATCHDOG_S=20 NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,P2P
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 tests/mp_worker.py --g-inter 2 --g-data 1 --mb 2 --batch 8 --cfg tiny --out /tmp > gpurun_out/p2p_diag.log 2>&1
echo "exit $?" >> gpurun_out/p2p_diag.log
grep -E "axonn|Error|TIMEOUT|via|Channel 00" gpurun_out/p2p_diag.log | head -40
