for v in base "$@"; do
  if [ "$v" = base ]; then E=""; else E="CVSR_LIB=build/variants/$v.so"; fi
  for rep in 1 2; do
  env $E timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); b=d['roofline_bp_iteration']
print('$v', 'val %.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], 'cn %.3f'%d['roofline']['frac'], {k:round(v,2) for k,v in b['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
  done
done
