cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "decode" 2>&1 | tail -2
timeout 900 python tools/bench_kernels.py 2>&1 | head -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_grid_kernel -c 1 -o gpurun_out/prof_decode_r01b python tools/bench_kernels.py > gpurun_out/ncu12.log 2>&1; echo "ncu rc=$?"
