cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -v "^    " | tail -20 > gpurun_out/test21.txt; tail -2 gpurun_out/test21.txt
timeout 900 python tools/bench_kernels.py 2>&1 | tail -5
