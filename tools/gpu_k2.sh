cd $GRAFT_REPO_ROOT
TAG=${TAG:-k2}
AFAM_RENDER2_MINB=${TESTV:-3} timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -k "frame or config3 or config2" -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
for r in 1 2; do
for v in $VARIANTS; do
  AFAM_RENDER2_MINB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-extra --steps 20 > gpurun_out/ab_${TAG}_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_${TAG}_$v.json')); print('$v', 'kernel_ms %.4f'%d['config']['kernel_ms'], 'value %.4e'%d['value'])"
done; done
if [ -n "$NCU" ]; then AFAM_RENDER2_MINB=$NCU timeout 900 ncu --set full --clock-control none --import-source on -k regex:render -s 3 -c 1 -o gpurun_out/prof_render_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/ncu_render_$TAG.log 2>&1; echo "ncu rc=$?"; fi
