# K3 iteration: decode parity tests, config-5 timing A/B, optional ncu
cd $GRAFT_REPO_ROOT
TAG=${TAG:-k3}
timeout 900 python -m pytest tests -m gpu -q -x -k "decode or config5 or grid" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
for v in ${VARIANTS:-x}; do echo "variant $v"; env $(echo $v | tr ',' ' ') timeout 300 python tools/bench_kernels.py 2>&1 | head -1; done
if [ -n "$NCU" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_fx -c 1 -o gpurun_out/prof_fx_$TAG python tools/bench_kernels.py > gpurun_out/ncu_fx_$TAG.log 2>&1; echo "ncu rc=$?"; fi
