cd $GRAFT_REPO_ROOT
timeout 2400 python tools/backoff.py --config C4 --frames 2000 > gpurun_out/t29_backoff.jsonl 2> gpurun_out/t29_backoff.err; echo "backoff rc $?"
python -c "
import json
for l in open('gpurun_out/t29_backoff.jsonl'):
    d=json.loads(l)
    if 'test' in d: print(d['slice'], d['family'], d['params'], d['test']['fer'], round(d['test']['mean_iters'],1), d['test']['undetected'], d['status'], '%.3g'%d['work'])
    else: print(d)
"
tail -3 gpurun_out/t29_backoff.err
