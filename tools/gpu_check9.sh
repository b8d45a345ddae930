cd $GRAFT_REPO_ROOT
timeout 600 python tools/diag_e2e.py > gpurun_out/diag_e2e.txt 2>&1; echo "diag rc=$?"
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo "bench rc=$?"
tail -2 gpurun_out/bench9.err
python -c "
import json; d=json.load(open('gpurun_out/bench9.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'cfg', {k: d['config'][k] for k in ('kernel_ms','host_envelope_ms','frame_ms')}, 'clocks', d['clocks'], 'roof', d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['shaded_frac'])
print('e2e', d['e2e'])"
grep -E "^(off|linear)" gpurun_out/diag_e2e.txt
