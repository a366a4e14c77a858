cd $GRAFT_REPO_ROOT
one() { timeout 300 env $1 python bench.py --no-e2e --no-cpu-baseline --no-other-schedule --steps 5 --warmup 3 ${@:2} 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*'.replace('build/variants/',''),'val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'layer_frac %.3f'%r['frac'],'fer',d['fer'],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
for c in C4 C4fast C3; do for v in base new skip6 minb5 skip6minb5; do one CVSR_LIB=build/variants/$v.so --config $c; done; done
