cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_pencil_kernel -c 1 -o gpurun_out/prof_decode_pencil python tools/bench_kernels.py > /dev/null 2>&1; echo "ncu rc=$?"
AFAM_DECODE_VARIANT=plane timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_grid_kernel -c 1 -o gpurun_out/prof_decode_plane python tools/bench_kernels.py > /dev/null 2>&1; echo "ncu rc=$?"
