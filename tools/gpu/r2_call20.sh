cd $GRAFT_REPO_ROOT
one() { timeout 300 env $1 python bench.py --no-e2e --no-cpu-baseline --no-other-schedule --steps 5 --warmup 3 ${@:2} 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*'.replace('build/variants/',''),'val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'layer_frac %.3f'%r['frac'],'iter_frac %.3f'%b['frac'],'fer',d['fer'],'beta %.4f'%d['beta'],[round(x,2) for x in d['mean_iters']],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()}, r['launches_per_step'])" || tail -3 gpurun_out/ab_err.txt; }
one CVSR_X=0
one CVSR_LAYER_RUNS=0
one CVSR_X=0 --config C2
one CVSR_LAYER_RUNS=0 --config C2
timeout 900 python -m pytest tests -m gpu -x -q -k "layered or reconcile" > gpurun_out/t20_layered.log 2>&1; echo "layered rc $?"; tail -2 gpurun_out/t20_layered.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_tma<.int.6, .int.2, .bool.1" -s 30 -c 1 -o gpurun_out/t20_l6 python tools/one_step.py --config C4 > gpurun_out/t20_ncu6.log 2>&1; echo "ncu6 rc $?"
