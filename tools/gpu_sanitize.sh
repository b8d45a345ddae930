# compute-sanitizer runs of the K1/K2/K3 paths and the replay (summaries under gpurun_out/)
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool workload
  timeout 1200 $CS --tool $1 --print-limit 20 python tools/sanitize.py $2 > gpurun_out/san_$1_$2.log 2>&1
  echo "$1 $2 rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard|ok$' gpurun_out/san_$1_$2.log | tr '\n' ' ' | cut -c1-200)"
}
run memcheck decode; run racecheck decode; run synccheck decode
run memcheck render; run racecheck render
run memcheck eval; run racecheck eval
run memcheck replay
run memcheck highdeg; run racecheck highdeg
# the IPC peer-store path: two processes render into rank 0's frame (tests/test_tiles_fused_gpu.py),
# and the two-frames-in-flight replay
timeout 1200 $CS --tool memcheck --target-processes all --print-limit 20 python -m pytest -q tests/test_tiles_fused_gpu.py > gpurun_out/san_memcheck_fused.log 2>&1
echo "memcheck fused rc=$? : $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_memcheck_fused.log | tr '\n' ' ' | cut -c1-300)"
timeout 1200 $CS --tool racecheck --target-processes all --print-limit 20 python -m pytest -q tests/test_tiles_fused_gpu.py > gpurun_out/san_racecheck_fused.log 2>&1
echo "racecheck fused rc=$? : $(grep -E 'RACECHECK SUMMARY|passed|failed' gpurun_out/san_racecheck_fused.log | tr '\n' ' ' | cut -c1-300)"
