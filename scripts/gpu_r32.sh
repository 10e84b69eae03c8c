set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python scripts/microbench.py --what adam > gpurun_out/adam_sweep.jsonl 2> gpurun_out/adam_sweep.err
bash scripts/gpu_prof.sh
