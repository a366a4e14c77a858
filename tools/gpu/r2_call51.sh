cd $GRAFT_REPO_ROOT
timeout 1500 python tools/sweep_nr.py > gpurun_out/t51_c5.jsonl 2> gpurun_out/t51_c5.err; echo "sweep rc $?"; tail -3 gpurun_out/t51_c5.jsonl | cut -c1-200
