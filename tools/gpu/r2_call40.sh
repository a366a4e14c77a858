cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_llr_interleaved" -s 3 -c 1 -o gpurun_out/t40_llr python tools/one_step.py --config C4 > gpurun_out/t40_ncu.log 2>&1; echo "ncu rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_synd_test" -s 20 -c 1 -o gpurun_out/t40_synd python tools/one_step.py --config C4 > gpurun_out/t40_ncu2.log 2>&1; echo "ncu2 rc $?"
