# Quick GPU check: full GPU test suite, then bench.py config-3 device value (no e2e / CPU leg / extras), twice.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-q}
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 ${PYTEST_ARGS} > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_$TAG.log
for r in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-extra --steps 20 > gpurun_out/b_$TAG.json 2>gpurun_out/b_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/b_$TAG.json')); print('kernel_ms %.4f'%d['config']['kernel_ms'], 'value %.4e'%d['value'], 'frac %.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/b_$TAG.err
done
