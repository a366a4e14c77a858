cd $GRAFT_REPO_ROOT
one() { timeout 300 env $1 python bench.py --no-e2e --no-cpu-baseline --no-other-schedule --steps 5 --warmup 3 ${@:2} 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*'.replace('build/variants/',''),'val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'layer_frac %.3f'%r['frac'],'fer',d['fer'],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
for r in 1 2; do for v in base ch3 ch6 w8 stage4; do one CVSR_LIB=build/variants/$v.so --config C4; done; done
for v in base ch3 ch6 w8 stage4; do one CVSR_LIB=build/variants/$v.so --config C4fast; done
