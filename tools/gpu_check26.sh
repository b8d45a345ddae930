cd $GRAFT_REPO_ROOT
TAG=new timeout 300 python tools/diag_k2.py 2>&1 | tail -6
TAG=old AFAM_LIB=$PWD/tools/ab/libafam_old.so timeout 300 python tools/diag_k2.py 2>&1 | tail -6
TAG=new_exact AFAM_RENDER_FORCE_EXACT=1 timeout 300 python tools/diag_k2.py 2>&1 | tail -6
