cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15
for m in 3 4; do AFAM_RENDER_MINB=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b23_$m.json 2>gpurun_out/b23_$m.err; python -c "
import json; d=json.load(open('gpurun_out/b23_$m.json')); print('MINB=$m value', d['value'], 'kernel_ms', d['config']['kernel_ms'], d['roofline'].get('shaded_frac'))"; done
