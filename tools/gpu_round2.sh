# Round-2 GPU session: parity tests, smoke, bench (ours + reference arm, all
# workloads), kernel microbenchmarks, ncu launch list and --set full captures
# of K2 (render2_kernel), K3 (decode) and K1 (points).  Outputs under gpurun_out/.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 600 python tools/bench_kernels.py > gpurun_out/kernels_$TAG.jsonl 2> gpurun_out/kernels_$TAG.err; echo "kernels rc=$?"
if [ -z "$NONCU" ]; then
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_ncu_$TAG.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render -s 3 -c 1 -o gpurun_out/prof_render_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/ncu_render_$TAG.log 2>&1; echo "ncu render rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode -c 1 -o gpurun_out/prof_decode_$TAG python tools/bench_kernels.py > gpurun_out/ncu_decode_$TAG.log 2>&1; echo "ncu decode rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:points -c 1 -o gpurun_out/prof_points_$TAG python tools/bench_kernels.py > gpurun_out/ncu_points_$TAG.log 2>&1; echo "ncu points rc=$?"
fi
head -c 4000 gpurun_out/bench_$TAG.json; echo; head -c 1500 gpurun_out/bench_ref_$TAG.json; echo; cut -c1-400 gpurun_out/kernels_$TAG.jsonl
