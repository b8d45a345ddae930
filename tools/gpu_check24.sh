cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_frames.py 2>&1 | tail -12
echo "--- force exact"
AFAM_RENDER_FORCE_EXACT=1 timeout 300 python tools/diag_frames.py 2>&1 | tail -12
