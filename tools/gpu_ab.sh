# bench (with the config-2 / config-5 extras) + K2 launch-bounds A/B
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02b}
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('c3', d['value'], d['config']['kernel_ms'])
for k,v in d.get('workloads',{}).items(): print(k, json.dumps(v)[:900])
"
for v in 3 4 5 3 4 5; do
  AFAM_RENDER2_MINB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-extra --steps 20 > gpurun_out/ab_${TAG}_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_${TAG}_$v.json')); print('MINB $v', 'kernel_ms %.4f'%d['config']['kernel_ms'], 'value %.4e'%d['value'])"
done
