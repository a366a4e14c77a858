cd $GRAFT_REPO_ROOT
one() { timeout 300 env $1 python bench.py --no-e2e --no-cpu-baseline --no-other-schedule --steps 5 --warmup 3 ${@:2} 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*','val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'layer_frac %.3f'%r['frac'],'fer',d['fer'],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
for c in C4 C2; do
for e in CVSR_COMPACT_FRAC=0.65 CVSR_COMPACT_FRAC=0.5 CVSR_COMPACT_FRAC=0.8 CVSR_COMPACT=0; do one $e --config $c; done
done
