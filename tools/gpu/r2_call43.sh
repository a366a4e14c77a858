cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_llr_interleaved" -s 1 -c 1 -o gpurun_out/t43_llr python tools/one_step.py --config C4 > gpurun_out/t43_ncu.log 2>&1; echo "ncu rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_compact_rows" -c 2 -o gpurun_out/t43_comp python tools/one_step.py --config C4 > gpurun_out/t43_ncu2.log 2>&1; echo "ncu2 rc $?"
