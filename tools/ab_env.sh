# A/B of environment switches on the default bench: each argument is one env assignment list
one() { timeout 300 env "$@" python bench.py --no-e2e --no-cpu-baseline 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*','val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'cn_frac %.3f'%r['frac'],'iter_frac %.3f'%b['frac'],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
for a in "$@"; do one $a; done
