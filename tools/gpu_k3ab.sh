# K3 A/B: decode parity tests on the in-tree build, then tools/bench_kernels.py's
# config-5 decode line for the in-tree build and each ab/*.so (swapped in), twice.
cd $GRAFT_REPO_ROOT
L=paper_2409_00184_b200/libafam.so
cp $L /tmp/libafam_main.so
timeout 900 python -m pytest tests -m gpu -q -k "decode or sharded" > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_k3.log
for v in /tmp/libafam_main.so ab/*.so; do
  cp $v $L
  for r in 1 2; do
    timeout 600 python tools/bench_kernels.py 2>/dev/null | grep "K3" | sed "s|^|$(basename $v) |" | cut -c1-200
  done
done
cp /tmp/libafam_main.so $L
