cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -v "^    " | tail -20 > gpurun_out/test18.txt; tail -2 gpurun_out/test18.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/bench18.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench18.json')); print('value', d['value'], 'kernel_ms', d['config']['kernel_ms'], d['roofline']['frac'])"
