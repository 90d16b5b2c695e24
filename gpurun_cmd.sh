cd $GRAFT_REPO_ROOT
python tools/phase_timing.py 4096 2>&1 | tail -16
