cd $GRAFT_REPO_ROOT
TAG=${TAG:-s11}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python tools/bench_kernels.py 2>&1 | head -1
AFAM_DECODE_FX_YPT=2 timeout 300 python tools/bench_kernels.py 2>&1 | head -1
timeout 900 python bench.py --workload config2 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/c2_$TAG.json 2>gpurun_out/c2_$TAG.err; echo "c2 rc=$?"; cut -c1-1500 gpurun_out/c2_$TAG.json
