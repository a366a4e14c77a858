# A/B of the CN kernels on the default bench (device-resident, no e2e / cpu baseline)
run() { timeout 300 env "$@" python bench.py --no-e2e --no-cpu-baseline 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*','val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'cn_frac %.3f'%r['frac'],'cn_us %.1f'%r['avg_launch_us'],'iter_frac %.3f'%b['frac'],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
run CVSR_CN_TMA=0
run CVSR_CN_TMA=1
run CVSR_CN_TMA=1 CVSR_CN_RING_KB=48
run CVSR_CN_TMA=1 CVSR_CN_RING_KB=72
run CVSR_CN_TMA=1 CVSR_CN_RING_KB=150
