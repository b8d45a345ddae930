cd $GRAFT_REPO_ROOT
for m in 3 4 5 6; do AFAM_RENDER_MINB=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b20_$m.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b20_$m.json')); print('MINB=$m value', d['value'], 'kernel_ms', d['config']['kernel_ms'])"; done
