cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_const.py > gpurun_out/diag_const.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench3a.json 2> gpurun_out/bench3a.err
timeout 600 env AFAM_NO_CLOCKS=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench3b.json 2> gpurun_out/bench3b.err
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15
cat gpurun_out/diag_const.txt | tail -30
python -c "
import json
for f in ('gpurun_out/bench3a.json','gpurun_out/bench3b.json'):
    try:
        d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['clocks'])
    except Exception as e: print(f, e)
"
tail -3 gpurun_out/bench3a.err
