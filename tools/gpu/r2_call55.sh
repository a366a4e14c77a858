cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/t55_bench.json 2> gpurun_out/t55_bench.err; echo "bench rc $?"
python -c "
import json; d=json.loads(open('gpurun_out/t55_bench.json').read().splitlines()[-1]); print('%.4g'%d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value'], d['clocks'])"
