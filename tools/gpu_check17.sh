cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 -o gpurun_out/prof_render_r01d python tools/prof_render.py --frames 3 --warm 1 > /dev/null 2>&1; echo "ncu rc=$?"
