cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/t10_bench.json 2> gpurun_out/t10_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/t10_ref.json 2> gpurun_out/t10_ref.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t10_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/t10_ncu.log 2>&1; echo "ncu list rc $?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:k_layer --csv --log-file gpurun_out/t10_traffic.csv python tools/one_step.py --config C4 > gpurun_out/t10_one_step.json 2> gpurun_out/t10_traffic.err; echo "ncu traffic rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.9" -s 6 -c 1 -o gpurun_out/t10_l9 python tools/one_step.py --config C4 > gpurun_out/t10_ncu9.log 2>&1; echo "ncu9 rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.7" -s 6 -c 1 -o gpurun_out/t10_l7 python tools/one_step.py --config C4 > gpurun_out/t10_ncu7.log 2>&1; echo "ncu7 rc $?"
CVSR_SUBS=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/t10_s1.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/t10_s1.json').read().splitlines()[-1]); print('S1', d['value'], d['ms_per_step'], d['roofline']['frac'])"
head -c 1500 gpurun_out/t10_bench.json
