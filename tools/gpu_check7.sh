cd $GRAFT_REPO_ROOT
for lib in libafam.so libafam_cache.so; do for m in 2 3 4; do echo "$lib MINB=$m"; AFAM_LIB=$PWD/paper_2409_00184_b200/$lib AFAM_RENDER_MINB=$m timeout 600 python tools/prof_render.py --frames 3,5,7,20,40 --warm 2 2>&1 | tail -5; done; done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -v "^    " | tail -40 > gpurun_out/test7.txt
tail -3 gpurun_out/test7.txt
