cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.6" -s 15 -c 1 -o gpurun_out/t70_l6 python tools/one_step.py --config C4 > gpurun_out/t70_ncu6.log 2>&1; echo "ncu6 rc $?"
