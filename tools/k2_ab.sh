# K2 A/B: GPU parity tests once, then bench.py (no e2e / CPU leg) under each
# VARIANTS entry ("NAME:ENV=V,ENV=V"), alternated twice.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-k2}
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
fi
for r in 1 2; do
for v in $VARIANTS; do
  name=${v%%:*}; envs=${v#*:}
  env $(echo $envs | tr ',' ' ') timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps ${STEPS:-20} > gpurun_out/ab_${TAG}_$name.json 2>gpurun_out/ab_${TAG}_$name.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${TAG}_$name.json')); print('$name', 'kernel_ms %.4f'%d['config']['kernel_ms'], 'value %.4e'%d['value'], 'frac %.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/ab_${TAG}_$name.err
done
done
