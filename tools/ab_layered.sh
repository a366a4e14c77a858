# A/B of k_layer variants on the default (layered) bench; args: variant names under build/variants
one() { timeout 300 env "$@" python bench.py --no-e2e --no-cpu-baseline 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*'.replace('build/variants/',''),'val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'layer_frac %.3f'%r['frac'],'iter_frac %.3f'%b['frac'],d['mean_iters'],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
one CVSR_SCHEDULE=layered
one CVSR_SUBS=2
for v in "$@"; do one CVSR_LIB=build/variants/$v.so; done
