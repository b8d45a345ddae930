cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_frames.py 2>&1 | tail -9
for m in 3 4 5; do AFAM_RENDER_MINB=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b25_$m.json 2>gpurun_out/b25_$m.err; python -c "
import json; d=json.load(open('gpurun_out/b25_$m.json')); print('MINB=$m value', d['value'], 'kernel_ms', d['config']['kernel_ms'], d['roofline'].get('shaded_frac'))"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/prof_render_r01f python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu rc=$?
