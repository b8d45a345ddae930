# A/B of libafam builds: GPU tests on the in-tree build, then bench.py's
# config-3 device value for the in-tree build and each ab/*.so (swapped in).
cd $GRAFT_REPO_ROOT
TAG=${TAG:-ab}
L=paper_2409_00184_b200/libafam.so
cp $L /tmp/libafam_main.so
if [ -z "$NOTEST" ]; then
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 ${PYTEST_ARGS} > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_$TAG.log
fi
for v in /tmp/libafam_main.so ab/*.so; do
  cp $v $L
  for r in 1 2; do
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-extra --steps 20 > gpurun_out/b_$TAG.json 2>gpurun_out/b_$TAG.err
    python -c "
import json; d=json.load(open('gpurun_out/b_$TAG.json')); print('$(basename $v)', 'kernel_ms %.4f'%d['config']['kernel_ms'], 'value %.4e'%d['value'], 'frac %.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/b_$TAG.err
  done
done
cp /tmp/libafam_main.so $L
