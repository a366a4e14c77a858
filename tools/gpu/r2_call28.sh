cd $GRAFT_REPO_ROOT
timeout 1800 python tools/try_s2.py --frames 1000 --rates 0.116 --core-rates 0.25,0.3,0.35,0.4,0.45 --no-met > gpurun_out/t28_s2.jsonl 2> gpurun_out/t28_s2.err; echo "rc $?"
cat gpurun_out/t28_s2.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['kind'], d['rate'], d['met'], 'fer', d['fer'], 'it %.1f'%d['mean_iters'], 'und', d['undetected'], 'dc', d['max_dc'], 'E', d['edges'], 's', d['seconds'])"
tail -3 gpurun_out/t28_s2.err
