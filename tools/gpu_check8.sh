cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -v "^    " | tail -30 > gpurun_out/test8.txt
tail -3 gpurun_out/test8.txt
for m in 3 4; do echo "MINB=$m"; AFAM_RENDER_MINB=$m timeout 600 python tools/prof_render.py --frames 3,5,7,20,40 --warm 2 2>&1 | tail -5; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench8.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'kernel_ms', d['config']['kernel_ms'], 'clocks', d['clocks'], 'frac', d['roofline']['frac'])
print('e2e', d['e2e'])"
