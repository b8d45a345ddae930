# K2 A/B: GPU parity tests, then bench with each launch-bounds variant, then an ncu capture.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-k2}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
for m in ${MINBS:-2 3 4}; do
  AFAM_RENDER_MINB=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b_${TAG}_$m.json 2>gpurun_out/b_${TAG}_$m.err
  python -c "
import json; d=json.load(open('gpurun_out/b_${TAG}_$m.json')); print('MINB=$m value %.3e'%d['value'], 'kernel_ms %.3f'%d['config']['kernel_ms'], 'frac %.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/b_${TAG}_$m.err
done
if [ -n "$NCU" ]; then
AFAM_RENDER_MINB=$NCU timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/prof_render_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_render_$TAG.log 2>&1; echo "ncu rc=$?"
fi
