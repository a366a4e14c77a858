cd $GRAFT_REPO_ROOT
one() { timeout 300 env $1 python bench.py --no-e2e --no-cpu-baseline --no-other-schedule --steps 5 --warmup 3 ${@:2} 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*'.replace('build/variants/',''),'val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'layer_frac %.3f'%r['frac'],'iter_frac %.3f'%b['frac'],'fer',d['fer'],'beta %.4f'%d['beta'],[round(x,2) for x in d['mean_iters']],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
one CVSR_X=0
one CVSR_LIB=build/variants/vload.so
one CVSR_X=0 --config C2
one CVSR_LIB=build/variants/vload.so --config C2
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/t11_other.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/t11_other.json').read().splitlines()[-1]); print('other', d.get('other_schedule'))"
timeout 1200 python tools/sweep_nr.py > gpurun_out/t11_c5.jsonl 2> gpurun_out/t11_c5.err; echo "sweep rc $?"; cat gpurun_out/t11_c5.jsonl | cut -c1-200
