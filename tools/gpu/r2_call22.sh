cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_layered.py -x -q -k "variants" > gpurun_out/t22_var.log 2>&1; echo "variants rc $?"; tail -15 gpurun_out/t22_var.log
