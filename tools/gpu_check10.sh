cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -v "^    " | tail -30 > gpurun_out/test10.txt
tail -3 gpurun_out/test10.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo "bench rc=$?"
tail -2 gpurun_out/bench10.err
python -c "
import json; d=json.load(open('gpurun_out/bench10.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'cfg', {k: d['config'][k] for k in ('kernel_ms','host_envelope_ms','frame_ms')}, 'clocks', d['clocks'], 'roof', d['roofline']['achieved'], d['roofline']['frac'])
print('e2e', d['e2e']); print('cpu', d.get('cpu_baseline'))"
