# A/B of library variants on one config: $1 = config, rest = variant names
cfg=$1; shift
one() { timeout 600 env "$@" python bench.py --config $cfg --no-e2e --no-cpu-baseline 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$cfg $*'.replace('build/variants/',''),'val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'cn_frac %.3f'%r['frac'],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
one CVSR_CN_TMA=0
for v in "$@"; do one CVSR_LIB=build/variants/$v.so; done
