# round-2: fused-kernel bottleneck probes; papers100m step launches; new tests; sanitizers
cd $GRAFT_REPO_ROOT
for c in papers100m mag240m products; do
  timeout 600 python tools/fused_bench.py --config $c --iters 20 --probe 0,1,2,4,3,5,6 >> gpurun_out/probe.jsonl 2>> gpurun_out/probe.err
done
cat gpurun_out/probe.jsonl
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size \
    --clock-control none --csv --log-file gpurun_out/launches_papers100m.csv \
    python tools/profile_step.py --config papers100m --steps 2 > gpurun_out/prof_p100m.log 2>&1
( time timeout 1800 python -m pytest -x -q tests/test_gpu_refsuite.py tests/test_gpu_ddp.py tests/test_gpu_codecs.py -s ) > gpurun_out/t_new.log 2>&1
tail -5 gpurun_out/t_new.log
( timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py ) > gpurun_out/sanitize_memcheck.log 2>&1
( timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_cases.py ) > gpurun_out/sanitize_racecheck.log 2>&1
( timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py ) > gpurun_out/sanitize_synccheck.log 2>&1
tail -3 gpurun_out/sanitize_*.log
