cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "decode or smoke" 2>&1 | tail -2
timeout 900 python tools/bench_kernels.py 2>&1 | head -1
