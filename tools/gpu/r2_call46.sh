cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -k "layered or reconcile" > gpurun_out/t46_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/t46_tests.log
one() { timeout 300 env $1 python bench.py --no-e2e --no-cpu-baseline --no-other-schedule --steps 5 --warmup 3 ${@:2} 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*','val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'layer_frac %.3f'%r['frac'],'fer',d['fer'],[round(x,2) for x in d['mean_iters']],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
for c in C4 C4fast C3 C2; do one CVSR_LAYER_PAIRS=0 --config $c; one CVSR_LAYER_PAIRS=1 --config $c; done
