cd $GRAFT_REPO_ROOT
timeout 900 python tools/e2e_probe.py papers100m 2>&1 | grep -v "^\[bench\]"
