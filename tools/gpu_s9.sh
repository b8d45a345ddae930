cd $GRAFT_REPO_ROOT
TAG=${TAG:-s9}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python tools/bench_kernels.py 2>&1 | cut -c1-200
AFAM_BENCH_SAME_GPU=1 AFAM_BENCH_BACKEND=gloo AFAM_NO_CLOCKS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 --no-extra --miss-load broadcast > gpurun_out/b2_bcast_$TAG.json 2> gpurun_out/b2_bcast_$TAG.err; echo "n2 bcast rc=$?"; tail -2 gpurun_out/b2_bcast_$TAG.err; cut -c1-400 gpurun_out/b2_bcast_$TAG.json; python -c "import json;d=json.load(open('gpurun_out/b2_bcast_$TAG.json'));print(d['e2e'])"
