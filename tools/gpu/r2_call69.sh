cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t69_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/t69_smoke.log
timeout 900 python bench.py > gpurun_out/t69_bench.json 2> gpurun_out/t69_bench.err; echo "bench rc $?"
for c in C4fast C2; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/t69_bench_$c.json 2> gpurun_out/t69_bench_$c.err; echo "bench $c rc $?"; done
python - <<'PY'
import json
for f in ["t69_bench.json","t69_bench_C4fast.json","t69_bench_C2.json"]:
    d=json.loads(open("gpurun_out/"+f).read().splitlines()[-1])
    print(f, "%.4g"%d["value"], "%.2f ms"%d["ms_per_step"], "frac %.3f"%d["roofline"]["frac"], "fer", d["fer"], "beta %.4f"%d["beta"], "e2e %.4g"%d["e2e"]["value"], d.get("other_schedule",{}).get("ms_per_step"), d["clocks"])
PY
