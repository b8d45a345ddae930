set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
