cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -v "^    " | tail -40 > gpurun_out/test6.txt
tail -3 gpurun_out/test6.txt
for m in 2 3; do echo "MINB=$m"; AFAM_RENDER_MINB=$m timeout 600 python tools/prof_render.py --frames 3,4,5,6,7 --warm 2 2>&1 | tail -5; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 -o gpurun_out/prof_render_r01c python tools/prof_render.py --frames 7 --warm 1 > gpurun_out/ncu6.log 2>&1; echo ncu rc=$?
