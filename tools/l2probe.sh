for F in 32 64 128 256 512 2048; do
  for S in 1 2 4; do
    if [ $F -lt $((32*S)) ]; then continue; fi
    CVSR_SUBS=$S CVSR_COMPACT=0 python bench.py --frames $F --no-e2e --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']; b=d['roofline_bp_iteration']
print($F,$S,'val %.3g'%d['value'],'ms %.2f'%d['ms_per_step'],'cn_GBs %.0f'%r['achieved'],'cn_us %.1f'%r['avg_launch_us'],'iter_GBs %.0f'%b['achieved'],b['kernel_ms_per_step'])"
  done
done
