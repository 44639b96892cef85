cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/sanitize.sh > gpurun_out/r2m_sanitize.log 2>&1
