cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t62_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t62_tests.log
one() { timeout 300 env $1 python bench.py --no-e2e --no-cpu-baseline --no-other-schedule --steps 5 --warmup 3 ${@:2} 2>gpurun_out/ab_err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print('$*'.replace('build/variants/',''),'val %.4g'%d['value'],'ms %.2f'%d['ms_per_step'],'layer_frac %.3f'%r['frac'],'fer',d['fer'],{k:round(v,2) for k,v in b['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_err.txt; }
for c in C4 C4fast C2 C3 C4b; do for v in base new; do one CVSR_LIB=build/variants/$v.so --config $c; done; done
