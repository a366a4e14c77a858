cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/t68_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t68_tests.log
