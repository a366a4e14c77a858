cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_llr_interleaved" -c 3 -o gpurun_out/t49_llr python tools/one_step.py --config C4 > gpurun_out/t49_ncu.log 2>&1; echo "ncu rc $?"
