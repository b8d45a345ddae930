# ncu captures of the current K2 (render), K3 (decode) and K1 (points) kernels + kernel microbenchmarks.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02a}
timeout 600 python tools/bench_kernels.py > gpurun_out/kernels_$TAG.jsonl 2> gpurun_out/kernels_$TAG.err; echo "kernels rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render -s 3 -c 1 -o gpurun_out/prof_render_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_render_$TAG.log 2>&1; echo "ncu render rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_grid_kernel -c 1 -o gpurun_out/prof_decode_$TAG python tools/bench_kernels.py > gpurun_out/ncu_decode_$TAG.log 2>&1; echo "ncu decode rc=$?"
cat gpurun_out/kernels_$TAG.jsonl
