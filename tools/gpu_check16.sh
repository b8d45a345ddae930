cd $GRAFT_REPO_ROOT
AFAM_BENCH_SAME_GPU=1 AFAM_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 1 > gpurun_out/bench16_n2.json 2> gpurun_out/bench16_n2.err; echo "n2 rc=$?"
tail -3 gpurun_out/bench16_n2.err; cat gpurun_out/bench16_n2.json | head -c 600; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench16_ref2.json 2>/dev/null; echo "ref2 rc=$?"; head -c 300 gpurun_out/bench16_ref2.json; echo
