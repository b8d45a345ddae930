# K2 A/B of two library builds (AFAM_LIB): the same bench config, alternated.
#   libafam_base.so (reference build) vs libafam.so (current)
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for lib in libafam_base.so libafam.so; do
  AFAM_LIB=$PWD/paper_2409_00184_b200/$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/ab_$lib.json 2>gpurun_out/ab_$lib.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$lib.json')); print('$lib', 'ms/frame %.4f'%d['ms_per_step'], 'value %.4e'%d['value'])" || tail -3 gpurun_out/ab_$lib.err
done
done
