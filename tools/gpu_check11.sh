cd $GRAFT_REPO_ROOT
timeout 900 python tools/bench_kernels.py 2>&1 | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_grid_kernel -c 1 -o gpurun_out/prof_decode_r01 python tools/bench_kernels.py > gpurun_out/ncu11.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench11.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench11.json')); print(d['value'], d['config']['host_envelope_ms'], d['e2e']['value'], d['e2e']['mean_rendering_ms'])"
