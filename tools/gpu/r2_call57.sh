cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "variants_bit_identical or layered_decode_parity or reconcile_layered" > gpurun_out/t57_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/t57_tests.log
