cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/t48_gpu.log 2>&1; echo "gpu tests rc $?"; tail -2 gpurun_out/t48_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t48_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/t48_smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/t48_ref.json 2> gpurun_out/t48_ref.err; echo "ref rc $?"
timeout 900 python bench.py > gpurun_out/t48_bench.json 2> gpurun_out/t48_bench.err; echo "bench rc $?"
for c in C4fast C2 C4b C3; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/t48_bench_$c.json 2> gpurun_out/t48_bench_$c.err; echo "bench $c rc $?"; done
python - <<'PY'
import json
for f in ["t48_bench.json","t48_bench_C4fast.json","t48_bench_C2.json","t48_bench_C4b.json","t48_bench_C3.json"]:
    try:
        d=json.loads(open("gpurun_out/"+f).read().splitlines()[-1])
        print(f, "%.4g"%d["value"], "%.2f ms"%d["ms_per_step"], "frac %.3f"%d["roofline"]["frac"], "fer", d["fer"], "beta %.4f"%d["beta"], "e2e %.4g"%d["e2e"]["value"] if d.get("e2e") else None, d.get("other_schedule",{}).get("ms_per_step"))
    except Exception as e: print(f, "ERR", e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t48_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-schedule > gpurun_out/t48_ncu.log 2>&1; echo "ncu list rc $?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:k_layer_tma --csv --log-file gpurun_out/t48_traffic.csv python tools/one_step.py --config C4 > gpurun_out/t48_one_step.json 2> gpurun_out/t48_traffic.err; echo "ncu traffic rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.7" -s 24 -c 1 -o gpurun_out/t48_l7 python tools/one_step.py --config C4 > gpurun_out/t48_ncu7.log 2>&1; echo "ncu7 rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.9" -s 24 -c 1 -o gpurun_out/t48_l9 python tools/one_step.py --config C4 > gpurun_out/t48_ncu9.log 2>&1; echo "ncu9 rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.6" -s 24 -c 1 -o gpurun_out/t48_l6 python tools/one_step.py --config C4 > gpurun_out/t48_ncu6.log 2>&1; echo "ncu6 rc $?"
