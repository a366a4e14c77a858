cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "hash or verify or session or smoke" > gpurun_out/t66_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t66_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t66_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/t66_smoke.log
one() { timeout 300 env $1 python bench.py --no-e2e --no-cpu-baseline --no-other-schedule --steps 5 --warmup 3 ${@:2} 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*','val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'fer',d['fer'],d['undetected_frames'],{k:round(v,3) for k,v in d['stage_ms_rank0'].items()})" || tail -3 gpurun_out/ab_err.txt; }
for c in C4 C2 C3; do one CVSR_X=1 --config $c; done
