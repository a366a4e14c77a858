set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -k "layered" > gpurun_out/t2_layered.log 2>&1; echo "layered rc $?"
tail -5 gpurun_out/t2_layered.log
for v in "" "CVSR_SUBS=2" "CVSR_LAYER_TMA=0"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/t2_bench_$(echo $v | tr '=' '_').json 2>&1; echo "bench [$v] rc $?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/t2_bench_$(echo $v | tr '=' '_').json').read().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['fer'])"
done
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/t2_bench_c2.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/t2_bench_c2.json').read().splitlines()[-1]); print('C2', d['value'], d['ms_per_step'], d['roofline']['frac'], d['fer'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer_tma -s 40 -c 3 -o gpurun_out/t2_layer_tma python tools/one_step.py --config C4 > gpurun_out/t2_ncu_full.log 2>&1; echo "ncu full rc $?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_layer --csv --log-file gpurun_out/t2_traffic.csv python tools/one_step.py --config C4 > gpurun_out/t2_one_step.json 2> gpurun_out/t2_traffic.err; echo "ncu traffic rc $?"
