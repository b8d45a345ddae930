cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_frames.py 2>&1 | tail -9
TAG=new timeout 300 python tools/diag_k2.py 2>&1 | tail -6
