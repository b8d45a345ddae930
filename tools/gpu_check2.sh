cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "eval_points or const or missing" 2>&1 | grep -v "^    " | head -150 > gpurun_out/fail2.txt
timeout 600 python tools/diag_render.py > gpurun_out/diag2.txt 2>&1
tail -30 gpurun_out/diag2.txt
