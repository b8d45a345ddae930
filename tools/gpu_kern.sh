# full GPU tests + kernel microbenchmarks (K3, K1) with optional A/B variants
cd $GRAFT_REPO_ROOT
TAG=${TAG:-kern}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for v in ${VARIANTS:-X=1}; do echo "variant $v"; env $(echo $v | tr ',' ' ') timeout 300 python tools/bench_kernels.py 2>&1 | cut -c1-250; done
