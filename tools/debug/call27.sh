cd "$GRAFT_REPO_ROOT"
bash tools/debug/call8.sh
bash tools/sanitize.sh > gpurun_out/sanitize.log 2>&1
