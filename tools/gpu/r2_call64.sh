cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t64_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/t64_smoke.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:k_layer_tma --csv --log-file gpurun_out/t64_traffic.csv python tools/one_step.py --config C4 > gpurun_out/t64_one_step.json 2> gpurun_out/t64_traffic.err; echo "ncu traffic rc $?"
python tools/ncu_traffic.py gpurun_out/t64_traffic.csv gpurun_out/t64_one_step.json --kernel k_layer_tma --algo-bytes 16 --out profiles/ncu_traffic_live.json && cp profiles/ncu_traffic_live.json gpurun_out/t64_traffic_live.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/t64_ref.json 2> gpurun_out/t64_ref.err; echo "ref rc $?"
timeout 900 python bench.py > gpurun_out/t64_bench.json 2> gpurun_out/t64_bench.err; echo "bench rc $?"
for c in C4fast C2 C4b C3; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/t64_bench_$c.json 2> gpurun_out/t64_bench_$c.err; echo "bench $c rc $?"; done
python - <<'PY'
import json
for f in ["t64_bench.json","t64_bench_C4fast.json","t64_bench_C2.json","t64_bench_C4b.json","t64_bench_C3.json"]:
    try:
        d=json.loads(open("gpurun_out/"+f).read().splitlines()[-1])
        print(f, "%.4g"%d["value"], "%.2f ms"%d["ms_per_step"], "frac %.3f"%d["roofline"]["frac"], "fer", d["fer"], "beta %.4f"%d["beta"], "e2e %.4g"%d["e2e"]["value"] if d.get("e2e") else None, d.get("other_schedule",{}).get("ms_per_step"), d["clocks"]["reasons"])
    except Exception as e: print(f, "ERR", e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t64_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-schedule > gpurun_out/t64_ncu.log 2>&1; echo "ncu list rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.7" -s 24 -c 1 -o gpurun_out/t64_l7 python tools/one_step.py --config C4 > gpurun_out/t64_ncu7.log 2>&1; echo "ncu7 rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.9" -s 24 -c 1 -o gpurun_out/t64_l9 python tools/one_step.py --config C4 > gpurun_out/t64_ncu9.log 2>&1; echo "ncu9 rc $?"
