for c in "$@"; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$c', '%.4g'%d['value'], '%.2f ms'%d['ms_per_step'], 'cn %.3f'%d['roofline']['frac'], {k:round(v,2) for k,v in d['roofline_bp_iteration']['kernel_ms_per_step'].items()})"; done
