set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -k "layered" > gpurun_out/t1_layered.log 2>&1; echo "layered rc $?"
timeout 1200 python -m pytest tests -m gpu -x -q -k "not layered" > gpurun_out/t1_rest.log 2>&1; echo "rest rc $?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t1_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/t1_bench.json 2> gpurun_out/t1_bench.err; echo "bench rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/t1_ncu.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/t1_layered.log gpurun_out/t1_rest.log gpurun_out/t1_smoke.log
cat gpurun_out/t1_bench.json | head -c 3000
